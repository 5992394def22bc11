#!/bin/bash
set -u
for sl in 0 256 1024; do
  if [ $sl = 0 ]; then F="-DHINM_TRACE"; else F="-DHINM_TRACE -DHINM_EPI_SLEEP=$sl"; fi
  HINM_EXP_FLAGS="$F" python -m paper_2407_20496_b200.build --experiments --force > /dev/null 2>&1
  cp scripts/libhinm_b200_exp.so scripts/libhinm_b200_sl$sl.so
  echo "== epi sleep $sl"
  HINM_B200_LIB=scripts/libhinm_b200_sl$sl.so timeout 300 python scripts/pair_trace.py 11008 4096 16384 2>&1 | head -13
  HINM_B200_LIB=scripts/libhinm_b200_sl$sl.so timeout 300 python scripts/pair_time.py 16384 up,down 2>&1 | cut -c1-160
done
