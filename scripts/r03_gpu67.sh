#!/bin/bash
# score kernel CTA width: 128 / 256 / 512 threads (whole 8 KB rows per CTA at 512 on the up projection)
set -u
for nt in 128 256 512 128 512; do
  echo "== NT $nt"; HINM_SCORES_NT=$nt HINM_B200_LIB=scripts/libhinm_b200_exp.so timeout 300 python scripts/compress_time.py 20 2>&1 | tail -1 | python3 -c "import json,sys; d=json.load(sys.stdin); print({k:(v['gpu_ms'],v['graph_matches_eager']) for k,v in d.items()})"
done
for nt in 128 512; do for sh in up down; do
  HINM_SCORES_NT=$nt HINM_B200_LIB=scripts/libhinm_b200_exp.so timeout 300 ncu --clock-control none --metrics gpu__time_duration.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed -k regex:k_scores8 --csv python scripts/compress_once.py $sh 2>/dev/null | tail -2 | awk -F'","' -v nt=$nt -v sh=$sh '{print nt, sh, $(NF-2), $NF}'
done; done
