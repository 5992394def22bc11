#!/bin/bash
# Round-2 GPU session 3: full GPU tests (image / saliency / bench-step / OCP), compressor timing + launch list.
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
echo "== pytest -m gpu"; timeout 1800 python -m pytest tests -q -m gpu 2>&1 | tail -25
echo "== compress time"; timeout 300 python scripts/compress_time.py 10 2>&1 | tail -2
echo "== ncu compress launch list"; timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_compress_r02.csv python scripts/compress_time.py 2 > /dev/null 2>&1; echo rc=$?
echo "== gyro timing (cfg1 default budgets)"; timeout 900 python scripts/gyro_time.py 768 3072 20 2>&1 | tail -2
