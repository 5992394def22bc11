#!/bin/bash
# the A path: 9 = 9/16 of the A bytes, 10 = no metadata copies, 11 = A split per MMA step, 4 = no A path (garbage results)
set -u
python -m paper_2407_20496_b200.build --experiments --force > /dev/null 2>&1
for d in 0 10 11 4 0; do echo "== dbg $d"; HINM_PAIR_DBG=$d HINM_B200_LIB=scripts/libhinm_b200_exp.so timeout 300 python scripts/pair_time.py 16384 up,down 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l); print(d['shape'], 'groups', d['groups_ms'])
    except Exception: print(l.strip()[:200])
"; done
