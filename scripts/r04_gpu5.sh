#!/bin/bash
# Round-2 fifth session: staggered compress_layers (hinm_compress_bf16_staged).
set -u
echo "== pytest"; timeout 600 python -m pytest tests/test_gpu_compress_layers.py tests/test_capi.py -q -x 2>&1 | tail -3
python scripts/layers_streams_ab.py
python scripts/compress_host_profile.py 2>&1 | sed -n 3,4p
