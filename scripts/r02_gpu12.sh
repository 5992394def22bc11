#!/bin/bash
# compressor rework check: GPU suite (compressor parity) + timing + launch list
set -u
mkdir -p gpurun_out
echo "== pytest -m gpu"; timeout 1800 python -m pytest tests -q -m gpu -x 2>&1 | tail -8
echo "== compress time"; timeout 300 python scripts/compress_time.py 10 2>&1 | tail -1
echo "== ncu compress launch list"; timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_compress_r02g.csv python scripts/compress_time.py 2 > /dev/null 2>&1; echo rc=$?
python scripts/launch_summary.py gpurun_out/launches_compress_r02g.csv gpurun_out/launches_compress_r02g.txt; head -30 gpurun_out/launches_compress_r02g.txt
