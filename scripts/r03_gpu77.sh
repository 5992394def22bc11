#!/bin/bash
# per-rank workload of the strong-scaling run on one GPU: 16384 global tokens over N = 1, 2, 4, 8 ranks
set -u
for t in 16384 8192 4096 2048; do
  timeout 600 python bench.py --tokens $t --no-cpu-baseline --no-extras 2>/dev/null | tail -1 | python3 -c "
import json,sys; d=json.loads(sys.stdin.read()); print($t, d['ms_per_step'], d['value'], d['speedup_vs_cublas'], d['per_spmm_image'])"
done
