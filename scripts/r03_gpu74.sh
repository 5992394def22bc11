#!/bin/bash
set -u
for bn in 128 256; do HINM_BN=$bn timeout 900 python scripts/bnt_sweep.py 2>&1 | grep "^{" > gpurun_out/bnt_$bn.jsonl; done
timeout 900 python scripts/bnt_sweep.py 2>&1 | grep "^{" > gpurun_out/bnt_auto.jsonl
wc -l gpurun_out/bnt_*.jsonl
