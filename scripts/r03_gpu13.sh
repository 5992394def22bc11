#!/bin/bash
set -u
HINM_EXP_FLAGS="-DHINM_TRACE" python -m paper_2407_20496_b200.build --experiments --force > /dev/null 2>&1
for im in groups tiles; do HINM_B200_LIB=scripts/libhinm_b200_exp.so timeout 300 python scripts/pair_utrace.py 11008 4096 16384 $im 2>&1 | tail -3; done
HINM_B200_LIB=scripts/libhinm_b200_exp.so timeout 300 python scripts/pair_utrace.py 4096 11008 16384 groups 2>&1 | tail -3
