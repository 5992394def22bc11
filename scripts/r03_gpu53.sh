#!/bin/bash
# compressor PDL chain: GPU suite on the default build, then compress timing with PDL on / off
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
for pdl in 1 0 1 0; do
  echo "== HINM_COMPRESS_PDL=$pdl"
  HINM_COMPRESS_PDL=$pdl HINM_B200_LIB=scripts/libhinm_b200_exp.so timeout 300 python scripts/compress_time.py 20 2>&1 | tail -3
done
