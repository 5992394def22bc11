#!/bin/bash
# early weight streams (default now): GPU suite, smoke, BERT / cfg1 configs, bench line
set -u
echo "== pytest -m gpu"; timeout 1800 python -m pytest tests -q -m gpu 2>&1 | tail -2
echo "== smoke"; timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for c in cfg1 cfg2; do timeout 300 python bench.py --config $c 2>/dev/null | python -c "
import sys,json
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['metric'], d['ms_per_step'], d['cublas_ms_per_step'], d['speedup_vs_cublas'])"; done
echo "== bench"; timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_r02i.json 2> gpurun_out/bench_r02i.err; echo rc=$?
