#!/bin/bash
set -u
mkdir -p gpurun_out
echo "== pytest compressor parity"; timeout 1200 python -m pytest tests -q -m gpu -x -k "parity or image or saliency or compress or next or gyro" 2>&1 | tail -3
echo "== compress time"; timeout 300 python scripts/compress_time.py 10 2>&1 | tail -1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_select_pack2|k_scores8" -c 10 -o gpurun_out/prof_comp6 python scripts/compress_time.py 1 > gpurun_out/prof_comp6.log 2>&1; echo rc=$?
