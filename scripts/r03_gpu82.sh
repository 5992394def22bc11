#!/bin/bash
# budget-select grid: CTAs = min(SMs / div, keys / per-CTA keys)
set -u
for cfg in "4 4096" "8 4096" "2 4096" "1 2048" "4 4096" "2 2048"; do
  set -- $cfg
  echo "== div $1 keys $2"; HINM_BSEL_DIV=$1 HINM_BSEL_KEYS=$2 HINM_B200_LIB=scripts/libhinm_b200_exp.so timeout 300 python scripts/compress_time.py 20 2>&1 | tail -1 | python3 -c "import json,sys; d=json.load(sys.stdin); print({k:(v['gpu_ms'],v['graph_matches_eager']) for k,v in d.items()})"
done
