#!/bin/bash
set -u
for ns in 4 6; do
  HINM_EXP_FLAGS="-DHINM_CHAIN_SLOTS=$ns" python -m paper_2407_20496_b200.build --experiments --force > /dev/null 2>&1
  echo "== slots $ns"; HINM_B200_LIB=scripts/libhinm_b200_exp.so timeout 300 python scripts/e2e_sweep.py 2>&1 | tail -1
done
