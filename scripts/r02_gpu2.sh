#!/bin/bash
# Round-2 GPU session 2: full GPU tests, new bench (both arms), gather-mechanism table, ncu evidence.
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
echo "== pytest -m gpu"; timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -15
echo "== smoke"; timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
echo "== bench N=1"; timeout 900 python bench.py > gpurun_out/bench_r02b.json 2> gpurun_out/bench_r02b.err; tail -c 4000 gpurun_out/bench_r02b.json; tail -3 gpurun_out/bench_r02b.err
echo "== bench reference"; (time timeout 900 python bench.py --impl reference --steps 5 --warmup 1) > gpurun_out/bench_ref_r02b.json 2>&1; tail -5 gpurun_out/bench_ref_r02b.json
echo "== gather mechanisms"; timeout 600 scripts/bin/gather_mechanisms > gpurun_out/gather_mechanisms_v2.txt 2>&1; echo rc=$?
echo "== ncu full spmm"; timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_hinm_spmm -s 10 -c 1 -o gpurun_out/prof_spmm_r02 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extras > gpurun_out/ncu_spmm.log 2>&1; echo rc=$?
echo "== ncu launch list"; timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r02.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extras > /dev/null 2>&1; echo rc=$?
