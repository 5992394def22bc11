#!/bin/bash
# Round-2 experiment: where does the up projection's per-unit time go? (experiments build)
set -u
mkdir -p gpurun_out
python -m paper_2407_20496_b200.build >/dev/null 2>&1
python -m paper_2407_20496_b200.build --experiments >/dev/null 2>&1
L=scripts/libhinm_b200_exp.so
for v in "" "HINM_GATHER=dbg_noepi" "HINM_BN=128" "HINM_GATHER=dbg_nomma" "HINM_GATHER=dbg_nogather" "HINM_GW=16"; do
  echo "== $v"; env HINM_B200_LIB=$L $v timeout 120 python scripts/spmm_time.py 16384 2>&1 | tail -1
done
