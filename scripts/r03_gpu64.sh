#!/bin/bash
# union-group first fit with register-resident list state vs the shared-memory list: same image, time
set -u
mkdir -p gpurun_out
timeout 600 python scripts/group_greedy_ab.py /tmp/new.npz 2>&1 | tail -3
HINM_GREEDY_SMEM=1 HINM_B200_LIB=scripts/libhinm_b200_exp.so timeout 600 python scripts/group_greedy_ab.py /tmp/old.npz 2>&1 | tail -3
python scripts/group_greedy_ab.py --cmp /tmp/new.npz /tmp/old.npz
timeout 600 python -m pytest tests/test_gpu_group.py tests/test_gpu_chain.py tests/test_gpu_shard.py -x -q 2>&1 | tail -1
timeout 600 ncu --clock-control none --metrics gpu__time_duration.sum -k regex:'k_greedy' --csv python scripts/group_build_time.py 2>/dev/null | grep k_greedy | awk -F'","' '{print $NF}' | head -8
