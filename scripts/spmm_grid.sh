#!/bin/bash
# Kernel-configuration sweep (experiments): LLaMA FFN shapes and the 4096^2 V sweep under every
# (X-stage rows, gather warps) pair.  Run under gpurun from the repo root.
for ks in 64 128; do for gw in 8 16; do
  echo "== KS=$ks GW=$gw"
  HINM_KS=$ks HINM_GW=$gw timeout 300 python scripts/spmm_time.py 16384
  HINM_KS=$ks HINM_GW=$gw timeout 300 python scripts/spmm_vsweep.py 16384
done; done
