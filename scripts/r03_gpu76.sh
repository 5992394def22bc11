#!/bin/bash
# L2 priorities of the pair kernel's streams: activation gathers (X) and weight image (A)
set -u
for cfg in "0 0" "1 0" "0 1" "0 2" "1 1" "0 0"; do
  set -- $cfg
  HINM_EXP_FLAGS="-DHINM_X_POLICY=$1 -DHINM_A_POLICY=$2" python -m paper_2407_20496_b200.build --experiments --force > /dev/null 2>&1
  echo "== X $1 A $2"
  HINM_B200_LIB=scripts/libhinm_b200_exp.so timeout 300 python scripts/pair_time.py 16384 up,down 2>&1 | grep "^{" | python3 -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d.get('shape'), {k: v for k, v in d.items() if 'ms' in k})"
  HINM_B200_LIB=scripts/libhinm_b200_exp.so timeout 300 ncu --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum -k regex:k_hinm_spmm -c 3 --csv python scripts/pair_time.py 16384 up 2>/dev/null | grep -E "dram__bytes|gpu__time" | tail -3 | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
done
