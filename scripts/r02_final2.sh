#!/bin/bash
# Round-2 evidence (third session): tests, smoke, bench (both arms), configs, launch lists
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
echo "== pytest -m gpu"; timeout 1800 python -m pytest tests -q -m gpu 2>&1 | tail -3
echo "== smoke"; timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
echo "== bench N=1"; timeout 900 python bench.py > gpurun_out/bench_final2.json 2> gpurun_out/bench_final2.err; echo rc=$?; tail -c 600 gpurun_out/bench_final2.json
echo "== bench reference arm"; timeout 900 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/bench_ref_final2.json 2>&1; tail -1 gpurun_out/bench_ref_final2.json | cut -c1-300
echo "== configs"; rm -f gpurun_out/configs_final2.jsonl
for c in cfg1 cfg2 cfg4 cfg4_875 cfg5; do timeout 600 python bench.py --config $c >> gpurun_out/configs_final2.jsonl 2>> gpurun_out/configs_final2.err; done
python - <<'PY'
import json
for l in open("gpurun_out/configs_final2.jsonl"):
    d = json.loads(l); print(d["metric"], d["ms_per_step"], d["cublas_ms_per_step"], d["speedup_vs_cublas"])
PY
echo "== power"; timeout 300 python scripts/power_probe.py 2>&1 | tail -4
