#!/bin/bash
# Round-2 re-entry (third session): GPU suite + smoke + default bench line on HEAD.
set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
echo "== pytest -m gpu"; timeout 1800 python -m pytest tests -q -m gpu -x 2>&1 | tail -5
echo "== smoke"; timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
echo "== compress time"; timeout 300 python scripts/compress_time.py 10 2>&1 | tail -3
echo "== bench"; timeout 900 python bench.py > gpurun_out/bench_r02g.json 2> gpurun_out/bench_r02g.err; echo rc=$?; tail -c 4000 gpurun_out/bench_r02g.json
