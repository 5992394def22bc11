#!/bin/bash
# ncu --set full of the compressor's kernels (LLaMA up), source-level
set -u
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:'k_select_pack2|k_tile_rank|k_bsel|k_survivors_ord|k_scores8' \
  -o gpurun_out/prof_comp_r03 -f python scripts/compress_once.py up > gpurun_out/prof_comp_r03.log 2>&1
tail -3 gpurun_out/prof_comp_r03.log
