#!/bin/bash
# Round-2 evidence session: tests, smoke, bench (both arms), launch lists, ncu captures, sanitizer.
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
echo "== pytest -m gpu"; timeout 1800 python -m pytest tests -q -m gpu 2>&1 | tail -3
echo "== smoke"; timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
echo "== bench N=1"; timeout 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; tail -c 1500 gpurun_out/bench_final.json
echo "== bench reference arm"; timeout 900 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/bench_ref_final.json 2>&1; tail -1 gpurun_out/bench_ref_final.json
echo "== ncu launch list (bench)"; timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_final.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extras > /dev/null 2>&1; echo rc=$?
echo "== ncu full spmm (up)"; timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_hinm_spmm -s 10 -c 1 -o gpurun_out/prof_spmm_final python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extras > /dev/null 2>&1; echo rc=$?
echo "== ncu compress launch list"; timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_compress_final.csv python scripts/compress_time.py 2 > /dev/null 2>&1; echo rc=$?
echo "== ncu full (tile gains, select+pack)"; timeout 600 ncu --set full --clock-control none -k regex:"k_tile_gains|k_select_pack|k_budget_coop" -c 3 -o gpurun_out/prof_compress_final python scripts/compress_time.py 1 > /dev/null 2>&1; echo rc=$?
echo "== compress time"; timeout 300 python scripts/compress_time.py 10 > gpurun_out/compress_final.json 2>&1; cat gpurun_out/compress_final.json
for t in memcheck synccheck racecheck; do echo "== sanitizer $t"; timeout 900 compute-sanitizer --tool $t python scripts/sanitize_smoke.py 2>&1 | tail -2; done > gpurun_out/sanitizer_final.txt 2>&1; cat gpurun_out/sanitizer_final.txt
