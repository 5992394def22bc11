#!/bin/bash
# Round-2 fifth session: compress_layers with one allocation / one sigma upload / raw stream launches.
set -u
mkdir -p gpurun_out
echo "== pytest"; timeout 600 python -m pytest tests/test_gpu_compress_layers.py -q -x 2>&1 | tail -3
python scripts/compress_host_profile.py 2>&1 | head -5
echo "== bench"; timeout 900 python bench.py > gpurun_out/bench_r04c.json 2> gpurun_out/bench_r04c.err; echo rc=$?
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_r04c.json").read().strip().splitlines()[-1])
c = d["compressor"]
print({k: c[k] for k in ["gpu_ms", "hbm_frac_gpu", "layers_concurrent_gpu_ms", "hbm_frac_layers_concurrent",
                         "layers_concurrent_stream_ms", "hbm_frac_layers_concurrent_stream", "hbm_frac_stream"]})
print(d["value"], d["speedup_vs_cublas"], d["roofline"]["frac"])
PY
