#!/bin/bash
# rows per select + pack CTA: 16 (product) / 32 / 64 (experiments build)
set -u
for r in 16 32 64 16; do
  HINM_EXP_FLAGS="-DHINM_SP2_ROWS=$r" python -m paper_2407_20496_b200.build --experiments --force > /dev/null 2>&1
  echo "== rows $r"; HINM_B200_LIB=scripts/libhinm_b200_exp.so timeout 300 python scripts/compress_time.py 20 2>&1 | tail -1 | python3 -c "import json,sys; d=json.load(sys.stdin); print({k:(v['gpu_ms'],v['graph_matches_eager']) for k,v in d.items()})"
done
