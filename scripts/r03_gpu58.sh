#!/bin/bash
# select+pack rework: parity (compressor + operand image tests), timing, ncu of the kernel
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_image.py tests/test_gpu_bench_step.py -x -q 2>&1 | tail -2
for i in 1 2; do timeout 300 python scripts/compress_time.py 20 2>&1 | tail -1 | python3 -c "import json,sys; d=json.load(sys.stdin); print({k:(v['gpu_ms'],v['graph_matches_eager']) for k,v in d.items()})"; done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:'k_select_pack2' -o gpurun_out/prof_sp2_r03b -f python scripts/compress_once.py up > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:'k_select_pack2' -o gpurun_out/prof_sp2_r03b_down -f python scripts/compress_once.py down > /dev/null 2>&1
ls gpurun_out/
