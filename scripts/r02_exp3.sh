#!/bin/bash
# Round-2 experiment: token blocks interleaved in the unit order (HINM_GB), LLaMA 16k tokens.
set -u
python -m paper_2407_20496_b200.build >/dev/null 2>&1
for gb in 1 2 3 4 1 2; do echo "== HINM_GB=$gb"; HINM_GB=$gb timeout 120 python scripts/spmm_time.py 16384 2>&1 | tail -1; done
echo "== variants test"; HINM_GB=2 timeout 600 python -m pytest tests/test_gpu_bench_step.py tests/test_gpu_parity.py -q -x 2>&1 | tail -2
