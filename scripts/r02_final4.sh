#!/bin/bash
# Round-2 evidence (fourth session, final): tests, smoke, bench (both arms), configs, sanitizer, launch list
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
echo "== pytest -m gpu"; timeout 1800 python -m pytest tests -q -m gpu 2>&1 | tail -2
echo "== smoke"; timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
echo "== bench N=1"; timeout 900 python bench.py > gpurun_out/bench_final4.json 2> gpurun_out/bench_final4.err; echo rc=$?
echo "== bench reference arm"; timeout 900 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/bench_ref_final4.json 2>&1; tail -1 gpurun_out/bench_ref_final4.json | cut -c1-200
echo "== configs"; rm -f gpurun_out/configs_final4.jsonl
for c in cfg1 cfg2 cfg4 cfg4_875 cfg5; do timeout 600 python bench.py --config $c >> gpurun_out/configs_final4.jsonl 2>> gpurun_out/configs_final4.err; done
python - <<'PY'
import json
for l in open("gpurun_out/configs_final4.jsonl"):
    d = json.loads(l); print(d["metric"], d["ms_per_step"], d["cublas_ms_per_step"], d["speedup_vs_cublas"])
PY
echo "== ncu launch list"; timeout 900 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second --clock-control none --csv --log-file gpurun_out/launches_final4.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extras > /dev/null 2>&1; echo rc=$?
for t in memcheck synccheck; do echo "== sanitizer $t"; timeout 1200 compute-sanitizer --tool $t python scripts/sanitize_smoke.py 2>&1 | tail -2; done
echo "== ncu compressor (up, down)"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:'k_select_pack2|k_tile_rank|k_bsel|k_survivors_ord|k_scores8|k_pack_offsets' -o gpurun_out/prof_comp_final4 -f python scripts/compress_once.py up > /dev/null 2>&1; echo rc=$?
echo "== compress timing"; timeout 300 python scripts/compress_time.py 20 2>&1 | tail -1
