#!/bin/bash
set -u
mkdir -p gpurun_out
echo "== pytest -m gpu"; timeout 1800 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
echo "== compress time"; timeout 300 python scripts/compress_time.py 10 2>&1 | tail -1
echo "== sanitizer compress"; timeout 600 compute-sanitizer --tool memcheck python scripts/sanitize_smoke.py 2>&1 | tail -4
echo "== racecheck compress"; timeout 900 compute-sanitizer --tool racecheck python scripts/sanitize_smoke.py 2>&1 | tail -4
