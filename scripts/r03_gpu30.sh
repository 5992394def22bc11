#!/bin/bash
# upper bound for a deeper X ring: A / metadata loads skipped (HINM_PAIR_DBG=4, garbage results)
set -u
for st in 4 5 6; do
  HINM_EXP_FLAGS="-DHINM_PAIR_STAGES=$st" python -m paper_2407_20496_b200.build --experiments --force > /dev/null 2>&1
  cp scripts/libhinm_b200_exp.so scripts/lib_st$st.so
  for d in 0 4; do
    echo "== stages $st dbg $d"; HINM_PAIR_DBG=$d HINM_B200_LIB=scripts/lib_st$st.so timeout 300 python scripts/pair_time.py 16384 up,down 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l); print(d['shape'], 'groups', d['groups_ms'])
    except Exception: print(l.strip()[:200])
"
  done
done
