#!/bin/bash
set -u
HINM_EXP_FLAGS="-DHINM_TRACE" python -m paper_2407_20496_b200.build --experiments --force > /dev/null 2>&1
for d in 0 2; do
  echo "== pair dbg $d"
  HINM_PAIR_DBG=$d HINM_B200_LIB=scripts/libhinm_b200_exp.so timeout 300 python scripts/pair_trace.py 11008 4096 16384 2>&1 | head -13
done
timeout 300 python scripts/pair_time.py 16384 up,down,sq_v32 2>&1 | cut -c1-220
echo "== group tests"; timeout 900 python -m pytest tests/test_gpu_group.py -x -q 2>&1 | tail -2
