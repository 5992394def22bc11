#!/bin/bash
set -u
mkdir -p gpurun_out
python -m paper_2407_20496_b200.build >/dev/null 2>&1
echo "== spmm time"; for i in 1 2; do timeout 120 python scripts/spmm_time.py 16384; done
echo "== pytest -m gpu"; timeout 1800 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
