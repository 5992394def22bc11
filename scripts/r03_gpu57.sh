#!/bin/bash
# HostChain: copies split by rows over 1 / 2 / 4 copy streams per direction, 3 / 4 slots
set -u
for cfg in "1 3" "2 3" "4 3" "2 4" "4 4"; do
  set -- $cfg
  HINM_EXP_FLAGS="-DHINM_CHAIN_ENGINES=$1 -DHINM_CHAIN_SLOTS=$2" python -m paper_2407_20496_b200.build --experiments --force > /dev/null 2>&1
  echo "== engines $1 slots $2"; HINM_B200_LIB=scripts/libhinm_b200_exp.so timeout 300 python scripts/e2e_sweep.py 2>&1 | tail -1
  HINM_CHAIN_NOCOMPUTE=1 HINM_B200_LIB=scripts/libhinm_b200_exp.so timeout 300 python scripts/e2e_sweep.py 2>&1 | tail -1 | cut -c1-40,80-
done
