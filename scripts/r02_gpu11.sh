#!/bin/bash
# current compressor breakdown + default bench line
set -u
mkdir -p gpurun_out
echo "== compress time"; timeout 300 python scripts/compress_time.py 10 2>&1 | tail -1
echo "== ncu compress launch list"; timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_compress_r02e.csv python scripts/compress_time.py 2 > /dev/null 2>&1; echo rc=$?
python scripts/launch_summary.py gpurun_out/launches_compress_r02e.csv gpurun_out/launches_compress_r02e.txt; head -30 gpurun_out/launches_compress_r02e.txt
echo "== bench"; timeout 900 python bench.py > gpurun_out/bench_r02e.json 2> gpurun_out/bench_r02e.err; echo rc=$?; tail -c 3000 gpurun_out/bench_r02e.json
