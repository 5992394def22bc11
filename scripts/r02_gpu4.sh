#!/bin/bash
# Round-2 GPU session 4: compressor v2 parity + timing, secondary configs through bench.py --config.
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
echo "== pytest -m gpu (compressor / parity)"; timeout 1800 python -m pytest tests -q -m gpu -x 2>&1 | tail -4
echo "== compress time"; timeout 300 python scripts/compress_time.py 10 2>&1 | tail -2
echo "== ncu compress launch list"; timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_compress_r02b.csv python scripts/compress_time.py 2 > /dev/null 2>&1; echo rc=$?
for c in cfg1 cfg2 cfg5 cfg4 cfg4_875; do echo "== bench --config $c"; timeout 600 python bench.py --config $c --steps 20 --warmup 3 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; tail -c 600 gpurun_out/bench_$c.json; echo; done
