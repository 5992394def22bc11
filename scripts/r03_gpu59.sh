#!/bin/bash
# select+pack with uint16 survivor lists (3 CTAs / SM on up, 1-2 on down): parity, timing, slots 8 vs 4
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_image.py tests/test_gpu_bench_step.py tests/test_gpu_group.py -x -q 2>&1 | tail -2
for i in 1 2; do timeout 300 python scripts/compress_time.py 20 2>&1 | tail -1 | python3 -c "import json,sys; d=json.load(sys.stdin); print({k:(v['gpu_ms'],v['graph_matches_eager']) for k,v in d.items()})"; done
echo "== slots 4 (exp build)"
for i in 1 2; do HINM_SP2_SLOTS=4 HINM_B200_LIB=scripts/libhinm_b200_exp.so timeout 300 python scripts/compress_time.py 20 2>&1 | tail -1 | python3 -c "import json,sys; d=json.load(sys.stdin); print({k:(v['gpu_ms'],v['graph_matches_eager']) for k,v in d.items()})"; done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:'k_select_pack2' -o gpurun_out/prof_sp2_r03c -f python scripts/compress_once.py up > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:'k_select_pack2' -o gpurun_out/prof_sp2_r03c_down -f python scripts/compress_once.py down > /dev/null 2>&1
