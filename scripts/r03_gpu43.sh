#!/bin/bash
# weight streams before griddepcontrol.wait (experiments build) on the PDL-short shapes (cfg1, cfg2)
set -u
HINM_EXP_FLAGS="-DHINM_EARLY_WEIGHTS" python -m paper_2407_20496_b200.build --experiments --force > /dev/null 2>&1
for lib in paper_2407_20496_b200/libhinm_b200.so scripts/libhinm_b200_exp.so paper_2407_20496_b200/libhinm_b200.so scripts/libhinm_b200_exp.so; do
  for c in cfg1 cfg2; do
    echo "== $lib $c"; HINM_B200_LIB=$lib timeout 300 python bench.py --config $c 2>/dev/null | python -c "
import sys,json
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d['cublas_ms_per_step'], d['speedup_vs_cublas'], [(r['gemm'], r['image'], r['spmm_ms']) for r in d['rows']])"
  done
done
