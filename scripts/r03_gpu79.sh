#!/bin/bash
# select + pack: 32 rows per CTA when one CTA fills the SM (down projection)
set -u
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_image.py tests/test_gpu_ties.py tests/test_gpu_bench_step.py tests/test_gpu_stream_order.py tests/test_gpu_group.py -x -q 2>&1 | tail -1
for i in 1 2 3; do timeout 300 python scripts/compress_time.py 20 2>&1 | tail -1 | python3 -c "import json,sys; d=json.load(sys.stdin); print({k:(v['gpu_ms'],v['hbm_frac_gpu'],v['graph_matches_eager']) for k,v in d.items()})"; done
timeout 900 compute-sanitizer --tool memcheck python scripts/sanitize_smoke.py 2>&1 | tail -1
