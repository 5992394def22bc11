#!/bin/bash
# CTA-pair kernel: stage-size / gather-warp variants, then one ncu --set full capture
set -u
mkdir -p gpurun_out
for v in "HINM_PAIR_KS=128 HINM_PAIR_GW=8" "HINM_PAIR_KS=64 HINM_PAIR_GW=8" "HINM_PAIR_KS=128 HINM_PAIR_GW=16" "HINM_PAIR_KS=64 HINM_PAIR_GW=16"; do
  echo "== $v"; env $v timeout 300 python scripts/pair_time.py 16384 sq_v64,up 2>&1 | cut -c1-200
done
echo "== ncu"; timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_hinm_spmm -s 8 -c 1 -o gpurun_out/prof_pair_r03 python scripts/pair_time.py 16384 sq_v64 > gpurun_out/ncu_pair.log 2>&1; echo rc=$?; tail -3 gpurun_out/ncu_pair.log
