#!/bin/bash
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
echo "== pytest -m gpu"; timeout 1800 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
echo "== compress time"; timeout 300 python scripts/compress_time.py 10 2>&1 | tail -1
echo "== ncu compress launch list"; timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_compress_r02d.csv python scripts/compress_time.py 2 > /dev/null 2>&1; echo rc=$?
