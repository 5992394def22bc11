#!/bin/bash
# sanitizer over the smoke incl. the union-group image + CTA-pair kernel
set -u
mkdir -p gpurun_out
for t in memcheck synccheck racecheck; do echo "== sanitizer $t"; timeout 1200 compute-sanitizer --tool $t python scripts/sanitize_smoke.py 2>&1 | tail -4; done > gpurun_out/sanitizer_r02c.txt 2>&1; cat gpurun_out/sanitizer_r02c.txt
