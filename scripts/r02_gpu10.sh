#!/bin/bash
# re-entry check: GPU suite on HEAD + die-locality gather microbenchmark
set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
echo "== die locality"; timeout 300 scripts/bin/die_locality 2>&1 | tee gpurun_out/die_locality.txt
echo "== pytest -m gpu"; timeout 1800 python -m pytest tests -q -m gpu -x 2>&1 | tail -5
