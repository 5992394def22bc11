#!/bin/bash
set -u
echo "== group tests"; timeout 900 python -m pytest tests/test_gpu_group.py -x -q 2>&1 | tail -3
timeout 300 python scripts/pair_time.py 16384 up,down,sq_v32,sq_v64_k25 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l); print(d['shape'], 'tiles', d['tiles_ms'], 'groups', d['groups_ms'], 'cublas', d['cublas_ms'], 'x', d['speedup_groups'])
    except Exception: print(l.strip()[:300])
"
for st in 4 6; do
  HINM_EXP_FLAGS="-DHINM_PAIR_STAGES=$st" python -m paper_2407_20496_b200.build --experiments --force > /dev/null 2>&1
  echo "== stages $st"; HINM_B200_LIB=scripts/libhinm_b200_exp.so timeout 300 python scripts/pair_time.py 16384 up,down 2>&1 | cut -c1-150
done
