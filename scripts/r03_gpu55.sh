#!/bin/bash
# select+pack ring depth (CTAs per SM): HINM_SP2_SLOTS = 4 / 6 / 8 (experiments build)
set -u
for ns in 8 6 4 8 6 4; do
  echo "== slots $ns"
  HINM_SP2_SLOTS=$ns HINM_B200_LIB=scripts/libhinm_b200_exp.so timeout 300 python scripts/compress_time.py 20 2>&1 | tail -1 | python3 -c "import json,sys; d=json.load(sys.stdin); print({k:(v['gpu_ms'],v['graph_matches_eager']) for k,v in d.items()})"
done
