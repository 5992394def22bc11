#!/bin/bash
# CTA-pair kernel: X-ring depth (experiments builds with HINM_PAIR_STAGES = 3, 5)
set -u
mkdir -p gpurun_out
summ() { python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l); print(d['shape'], 'tiles', d['tiles_ms'], 'groups', d['groups_ms'], 'cublas', d['cublas_ms'], 'x_groups', d['speedup_groups'])
    except Exception: print(l.strip()[:300])
"; }
echo "== default (4)"; timeout 300 python scripts/pair_time.py 16384 up,down 2>&1 | summ
for st in 3 5; do
  HINM_EXP_FLAGS="-DHINM_PAIR_STAGES=$st" python -m paper_2407_20496_b200.build --experiments --force > /dev/null 2>&1
  cp scripts/libhinm_b200_exp.so scripts/libhinm_b200_st$st.so
  for gw in 8 16; do
    echo "== stages $st gw $gw"; HINM_B200_LIB=scripts/libhinm_b200_st$st.so HINM_PAIR_GW=$gw timeout 300 python scripts/pair_time.py 16384 up,down 2>&1 | summ
  done
done
