#!/bin/bash
# union-group image + CTA-pair kernel: parity tests, then timing
set -u
mkdir -p gpurun_out
echo "== group tests"; timeout 900 python -m pytest tests/test_gpu_group.py -x -q 2>&1 | tail -15
echo "== pair timing"; timeout 600 python scripts/pair_time.py 16384 2>&1 | tee gpurun_out/pair_time_r03a.txt
