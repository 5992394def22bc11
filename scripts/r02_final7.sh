#!/bin/bash
# Round-2 evidence refresh after the last compressor / group-build changes: GPU suite, smoke, bench, launch list
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
echo "== pytest -m gpu"; timeout 1800 python -m pytest tests -q -m gpu 2>&1 | tail -1
echo "== smoke"; timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
echo "== bench N=1"; timeout 900 python bench.py > gpurun_out/bench_final7.json 2> gpurun_out/bench_final7.err; echo rc=$?
echo "== ncu launch list"; timeout 900 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second --clock-control none --csv --log-file gpurun_out/launches_final7.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extras > /dev/null 2>&1; echo rc=$?
