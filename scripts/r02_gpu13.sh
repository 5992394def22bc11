#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_tile_rank -s 2 -c 2 -o gpurun_out/prof_rank python scripts/compress_time.py 1 > gpurun_out/prof_rank.log 2>&1; echo rc=$?
tail -3 gpurun_out/prof_rank.log
