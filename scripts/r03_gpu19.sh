#!/bin/bash
set -u
HINM_EXP_FLAGS="-DHINM_TRACE" python -m paper_2407_20496_b200.build --experiments --force > /dev/null 2>&1
for d in 0 3; do echo "== dbg $d"; HINM_PAIR_DBG=$d HINM_B200_LIB=scripts/libhinm_b200_exp.so timeout 300 python scripts/pair_trace.py 11008 4096 16384 2>&1 | head -9; done
