#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none -k regex:k_hinm_spmm -s 14 -c 1 -o gpurun_out/prof_bench_down_r02 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extras > gpurun_out/ncu_bench_down.log 2>&1; echo rc=$?
