#!/bin/bash
# what the per-unit gap is made of: no epilogue (3), drain without stores (12), release first then drain+stores (13)
set -u
for d in 0 12 14 0; do
  echo "== PAIR_DBG $d"
  if [ "$d" = "0" ]; then unset HINM_PAIR_DBG; else export HINM_PAIR_DBG=$d; fi
  HINM_B200_LIB=scripts/libhinm_b200_exp.so timeout 300 python scripts/pair_time.py 16384 up,down 2>&1 | grep "^{" | python3 -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d.get('shape'), d['groups_ms'])"
  HINM_B200_LIB=scripts/libhinm_b200_exp.so timeout 300 python scripts/power_variants.py scripts/libhinm_b200_exp.so 2>&1 | tail -1
done
