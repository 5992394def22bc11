#!/bin/bash
# One GPU session that produces the round's evidence (run under gpurun from the repo root).
# Outputs land in gpurun_out/ and are summarised into profiles/ by scripts/ncu_summary.py,
# scripts/launch_summary.py and scripts/traffic_json.py.
set -u
mkdir -p gpurun_out
python -m paper_2407_20496_b200.build
echo "== pytest -m gpu"; timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
echo "== smoke"; timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
echo "== bench N=1"; timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err; tail -1 gpurun_out/bench_n1.json
echo "== bench reference arm"; timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2>&1; tail -1 gpurun_out/bench_ref.json
echo "== configs"; timeout 900 python scripts/bench_configs.py > gpurun_out/configs.json 2> gpurun_out/configs.err; tail -2 gpurun_out/configs.err
echo "== ncu launch list"; timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo rc=$?
echo "== ncu full (spmm, up projection of the bench step)"; timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_hinm_spmm -s 10 -c 1 -o gpurun_out/prof_spmm_final python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo rc=$?
echo "== ncu full (compressor select+pack)"; timeout 600 ncu --set full --clock-control none -k regex:k_select_pack -s 1 -c 1 -o gpurun_out/prof_compress_final python scripts/compress_time.py 1 > /dev/null 2>&1; echo rc=$?
