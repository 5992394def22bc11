#!/bin/bash
set -u
HINM_EXP_FLAGS="-DHINM_SPREAD_ALL" python -m paper_2407_20496_b200.build --experiments --force > /dev/null 2>&1
echo "== default"; timeout 300 python scripts/pair_time.py 16384 2>&1 | cut -c1-250
echo "== spread all (1-SM kernel gather warps off the MMA sub-partition)"; HINM_B200_LIB=scripts/libhinm_b200_exp.so timeout 300 python scripts/pair_time.py 16384 up,down,sq_v64,sq_v64_k25 2>&1 | cut -c1-250
