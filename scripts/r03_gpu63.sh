#!/bin/bash
# select+pack: rotated group order per lane pair (default build) vs none (experiments build, HINM_SP2_SKEW=0)
set -u
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_image.py tests/test_gpu_ties.py tests/test_gpu_bench_step.py -x -q 2>&1 | tail -1
for i in 1 2; do
  echo "skew"; timeout 300 python scripts/compress_time.py 20 2>&1 | tail -1 | python3 -c "import json,sys; d=json.load(sys.stdin); print({k:(v['gpu_ms'],v['graph_matches_eager']) for k,v in d.items()})"
  echo "no skew"; HINM_B200_LIB=scripts/libhinm_b200_exp.so timeout 300 python scripts/compress_time.py 20 2>&1 | tail -1 | python3 -c "import json,sys; d=json.load(sys.stdin); print({k:(v['gpu_ms'],v['graph_matches_eager']) for k,v in d.items()})"
done
for sh in up down; do
  timeout 300 ncu --clock-control none --metrics gpu__time_duration.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,smsp__inst_executed.sum -k regex:k_select_pack2 --csv python scripts/compress_once.py $sh 2>/dev/null | tail -3 | awk -F'","' '{print $(NF-2), $NF}'
done
