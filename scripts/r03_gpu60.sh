#!/bin/bash
# score kernel: rows of loads in flight per thread (8 / 16 / 32), timing + ncu
set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
for rb in 8 16 32 16; do echo "== RB $rb"; HINM_SCORES_RB=$rb HINM_B200_LIB=scripts/libhinm_b200_exp.so timeout 300 python scripts/compress_time.py 20 2>&1 | tail -1 | python3 -c "import json,sys; d=json.load(sys.stdin); print({k:(v['gpu_ms'],v['graph_matches_eager']) for k,v in d.items()})"; done
for rb in 8 16 32; do HINM_SCORES_RB=$rb HINM_B200_LIB=scripts/libhinm_b200_exp.so timeout 300 ncu --metrics gpu__time_duration.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed -k regex:k_scores8 --csv python scripts/compress_once.py up 2>/dev/null | tail -2 | cut -c1-30,200-; done
