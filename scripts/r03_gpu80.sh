#!/bin/bash
set -u
for r in 16 8 32 16 8; do
  echo "== rows $r"; HINM_SP2_ROWS=$r HINM_B200_LIB=scripts/libhinm_b200_exp.so timeout 300 python scripts/compress_time.py 20 2>&1 | tail -1 | python3 -c "import json,sys; d=json.load(sys.stdin); print({k:(v['gpu_ms'],v['graph_matches_eager']) for k,v in d.items()})"
done
