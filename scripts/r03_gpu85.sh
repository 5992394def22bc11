#!/bin/bash
# L2 priority of the Y stores: evict_first (product) / evict_normal / evict_last
set -u
for yp in 0 1 2 0; do
  HINM_EXP_FLAGS="-DHINM_Y_POLICY=$yp" python -m paper_2407_20496_b200.build --experiments --force > /dev/null 2>&1
  echo "== Y policy $yp"
  HINM_B200_LIB=scripts/libhinm_b200_exp.so timeout 300 python scripts/pair_time.py 16384 up,down 2>&1 | grep "^{" | python3 -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d.get('shape'), d['groups_ms'], d['tiles_ms'])"
  timeout 300 python scripts/power_variants.py scripts/libhinm_b200_exp.so 2>&1 | tail -1
done
