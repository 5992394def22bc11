#!/bin/bash
# refitted per-call image choice: tests, bench configs
set -u
timeout 900 python -m pytest tests/test_gpu_group.py tests/test_gpu_chain.py tests/test_gpu_variants.py tests/test_gpu_bench_step.py -x -q 2>&1 | tail -1
rm -f gpurun_out/configs_r03c.jsonl
for c in cfg1 cfg2 cfg4 cfg4_875 cfg5; do timeout 600 python bench.py --config $c >> gpurun_out/configs_r03c.jsonl 2>> gpurun_out/configs_r03c.err; done
python3 - <<'PY'
import json
for l in open("gpurun_out/configs_r03c.jsonl"):
    d = json.loads(l); print(d["metric"], d["ms_per_step"], d["cublas_ms_per_step"], d["speedup_vs_cublas"])
PY
