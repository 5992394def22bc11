#!/bin/bash
set -u
mkdir -p gpurun_out
for v in "HINM_PAIR_KS=128 HINM_PAIR_GW=8" "HINM_PAIR_KS=64 HINM_PAIR_GW=8" "HINM_PAIR_KS=128 HINM_PAIR_GW=16"; do
  echo "== $v"; env $v timeout 300 python scripts/pair_time.py 16384 sq_v64,up,down 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l); print(d['shape'], 'tiles', d['tiles_ms'], 'groups', d['groups_ms'], 'cublas', d['cublas_ms'], 'x_groups', d['speedup_groups'])
    except Exception: print(l.strip()[:300])
"
done
echo "== group tests"; timeout 900 python -m pytest tests/test_gpu_group.py -x -q 2>&1 | tail -2
