#!/bin/bash
set -u
echo "== compressor parity"; timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_image.py -x -q 2>&1 | tail -2
echo "== compress time"; timeout 300 python scripts/compress_time.py 10 2>&1 | tail -2
