#!/bin/bash
set -u
mkdir -p gpurun_out
echo "== group tests"; timeout 900 python -m pytest tests/test_gpu_group.py -x -q 2>&1 | tail -2
rm -f gpurun_out/configs_r02d.jsonl
for c in cfg1 cfg2 cfg4 cfg5; do timeout 600 python bench.py --config $c >> gpurun_out/configs_r02d.jsonl 2>> gpurun_out/configs_r02d.err; done
python - <<'PY'
import json
for l in open("gpurun_out/configs_r02d.jsonl"):
    d = json.loads(l)
    print(d["metric"], d["ms_per_step"], d["cublas_ms_per_step"], d["speedup_vs_cublas"])
    for r in d["rows"]:
        print("   ", r["gemm"], r["image"], r["spmm_ms"], r["cublas_ms"], r["speedup"], r["count"])
PY
