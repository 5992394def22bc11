#!/bin/bash
# 2-SM sparse MMA probe + rate; compressor slow-call repro with a launch list
set -u
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -o scripts/bin/probe_2sm scripts/probe_2sm.cu 2>/dev/null
echo "== probe_2sm"; timeout 120 scripts/bin/probe_2sm 2>&1 | tee gpurun_out/probe_2sm.txt
echo "== compress repro"; timeout 300 python scripts/compress_bench_repro.py 3 2>&1 | tail -9
echo "== ncu compress repro"; timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_compress_repro.csv python scripts/compress_bench_repro.py 2 > /dev/null 2>&1; echo rc=$?
python scripts/launch_summary.py gpurun_out/launches_compress_repro.csv gpurun_out/launches_compress_repro.txt 2>&1 | tail -2; head -40 gpurun_out/launches_compress_repro.txt
