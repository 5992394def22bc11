#!/bin/bash
set -u
mkdir -p gpurun_out
for sl in 4 8 12 16; do
  echo "== slots $sl"
  HINM_SP2_SLOTS=$sl HINM_B200_LIB=scripts/libhinm_b200_exp.so timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_select_pack2 -c 4 python scripts/compress_time.py 1 2>&1 | grep -E "gpu__time_duration" | head -4
done
