#!/bin/bash
# Round-2 GPU session 1: baseline re-check + gather-mechanism / X-layout / TMEM-metadata experiments.
set -u
mkdir -p gpurun_out scripts/bin
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m paper_2407_20496_b200.build
python -m paper_2407_20496_b200.build --experiments
nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -o scripts/bin/gather_mechanisms scripts/gather_mechanisms.cu -lcuda
nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -o scripts/bin/probe_sparse_meta scripts/probe_sparse_meta.cu
echo "== probe"; timeout 60 scripts/bin/probe_sparse_meta > gpurun_out/probe_meta.txt 2>&1; echo rc=$?; head -5 gpurun_out/probe_meta.txt
echo "== gather mechanisms"; timeout 300 scripts/bin/gather_mechanisms > gpurun_out/gather_mechanisms.txt 2>&1; echo rc=$?; cat gpurun_out/gather_mechanisms.txt
echo "== xblk"
for x in 0 1 0 1; do HINM_B200_LIB=scripts/libhinm_b200_exp.so HINM_XBLK=$x timeout 120 python scripts/spmm_time.py 16384; done 2>&1 | tee gpurun_out/xblk.txt
for g in dbg_nomma dbg_nogather; do for x in 0 1; do HINM_B200_LIB=scripts/libhinm_b200_exp.so HINM_GATHER=$g HINM_XBLK=$x timeout 120 python scripts/spmm_time.py 16384; done; done 2>&1 | tee -a gpurun_out/xblk.txt
echo "== bench"; timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_r02a.json 2> gpurun_out/bench_r02a.err; tail -c 3000 gpurun_out/bench_r02a.json
echo "== pytest -m gpu"; timeout 1200 python -m pytest tests -x -q -m gpu 2>&1 | tail -5
