#!/bin/bash
# Round-2 fifth session: compress_layers parity + the bench line with the concurrent compressor.
set -u
mkdir -p gpurun_out
echo "== pytest compress_layers"; timeout 600 python -m pytest tests/test_gpu_compress_layers.py tests/test_bench_cpu.py -q -x 2>&1 | tail -3
echo "== bench"; timeout 900 python bench.py > gpurun_out/bench_r04a.json 2> gpurun_out/bench_r04a.err; echo rc=$?
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_r04a.json").read().strip().splitlines()[-1])
print(json.dumps(d["compressor"]))
print(d["value"], d["speedup_vs_cublas"], d["roofline"]["frac"])
PY
