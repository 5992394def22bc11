#!/bin/bash
# Round-2 GPU session 6: SpMM unit-boundary look-ahead, k-means distance fix: tests + timing.
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
echo "== pytest -m gpu"; timeout 1800 python -m pytest tests -q -m gpu 2>&1 | tail -4
echo "== spmm time"; for i in 1 2; do timeout 120 python scripts/spmm_time.py 16384; done
echo "== compress time"; timeout 300 python scripts/compress_time.py 10 2>&1 | tail -1
echo "== bench"; timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_r02f.json 2> gpurun_out/bench_r02f.err; python -c "
import json; d=json.loads(open('gpurun_out/bench_r02f.json').read().strip().splitlines()[-1]); print({k: d[k] for k in ('value','ms_per_step','speedup_vs_cublas','per_spmm_ms')}, d['roofline']['frac'], d['roofline']['binding'], d.get('v128'), d['compressor']['hbm_frac_stream'])"
