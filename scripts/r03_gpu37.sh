#!/bin/bash
# BERT cfg2 rows: per-tile 256- vs 128-token units vs union-group image (CUDA graphs)
set -u
for v in "HINM_GROUPS=0 HINM_BN=256" "HINM_GROUPS=0 HINM_BN=128" "HINM_GROUPS=1" ""; do
  echo "== $v"; env $v timeout 300 python bench.py --config cfg2 2>/dev/null | python -c "
import sys,json
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d['cublas_ms_per_step'], d['speedup_vs_cublas'], [(r['gemm'], r['image'], r['spmm_ms'], r['cublas_ms']) for r in d['rows']])"
done
