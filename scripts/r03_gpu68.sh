#!/bin/bash
# |bf16| -> fp64 by integer rebiasing (no F2F) in the score / select kernels: parity + timing + ncu
set -u
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_image.py tests/test_gpu_ties.py tests/test_gpu_bench_step.py tests/test_gpu_gyro.py -x -q 2>&1 | tail -1
for i in 1 2 3; do timeout 300 python scripts/compress_time.py 20 2>&1 | tail -1 | python3 -c "import json,sys; d=json.load(sys.stdin); print({k:(v['gpu_ms'],v['hbm_frac_gpu'],v['graph_matches_eager']) for k,v in d.items()})"; done
for sh in up down; do
  timeout 300 ncu --clock-control none --metrics gpu__time_duration.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed -k regex:k_scores8 --csv python scripts/compress_once.py $sh 2>/dev/null | tail -2 | awk -F'","' -v sh=$sh '{print sh, $(NF-2), $NF}'
done
