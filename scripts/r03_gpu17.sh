#!/bin/bash
set -u
mkdir -p gpurun_out
echo "== pytest -m gpu"; timeout 1800 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
echo "== bench"; timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_r03b.json 2> gpurun_out/bench_r03b.err; echo rc=$?; tail -3 gpurun_out/bench_r03b.err
