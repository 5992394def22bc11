#!/bin/bash
# ncu of the up-projection launch inside the bench step (pair kernel): DRAM / L2 / tensor metrics
set -u
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_hinm_spmm -s 13 -c 1 -o gpurun_out/prof_bench_up_r03 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extras > gpurun_out/ncu_bench.log 2>&1; echo rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,smsp__cycles_active.avg --clock-control none --csv --log-file gpurun_out/launches_bench_r03.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extras > /dev/null 2>&1; echo rc=$?
