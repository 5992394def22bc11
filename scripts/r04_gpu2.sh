#!/bin/bash
# Round-2 fifth session: host cost of compress after the carve / device-context changes, parity, bench.
set -u
mkdir -p gpurun_out
python scripts/compress_host_profile.py 2>&1 | head -4
echo "== pytest"; timeout 900 python -m pytest tests/test_gpu_compress_layers.py tests/test_gpu_parity.py tests/test_gpu_image.py tests/test_gpu_next.py tests/test_gpu_shard.py -q -x 2>&1 | tail -3
echo "== bench"; timeout 900 python bench.py > gpurun_out/bench_r04b.json 2> gpurun_out/bench_r04b.err; echo rc=$?
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_r04b.json").read().strip().splitlines()[-1])
print(json.dumps(d["compressor"]))
print(d["value"], d["speedup_vs_cublas"], d["roofline"]["frac"])
PY
