#!/bin/bash
set -u
mkdir -p gpurun_out
echo "== ncu pair"; timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_hinm_spmm -s 2 -c 1 -o gpurun_out/prof_pair_r03b python scripts/pair_only.py 4096 4096 64 0.5 16384 3 > gpurun_out/ncu_pair.log 2>&1; echo rc=$?; tail -2 gpurun_out/ncu_pair.log
