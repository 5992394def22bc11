#!/bin/bash
# Round-2 GPU session 5: select+pack staging, k-means distances on the GPU: tests + compressor timing.
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
echo "== pytest -m gpu"; timeout 1800 python -m pytest tests -q -m gpu -x 2>&1 | tail -4
for r in 8 4; do echo "== compress time HINM_SP_R=$r"; HINM_SP_R=$r timeout 300 python scripts/compress_time.py 10 2>&1 | tail -1; done
echo "== ncu compress launch list"; timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_compress_r02c.csv python scripts/compress_time.py 2 > /dev/null 2>&1; echo rc=$?
echo "== gyro timing (cfg1 default budgets)"; timeout 900 python scripts/gyro_time.py 768 3072 20 2>&1 | tail -1
