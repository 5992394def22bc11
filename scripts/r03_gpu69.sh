#!/bin/bash
# racecheck on the final compressor / group build / SpMM smoke, with and without the select+pack kernel
set -u
timeout 2400 compute-sanitizer --tool racecheck --racecheck-report hazard --kernel-name-exclude kns=k_select_pack2 python scripts/sanitize_smoke.py > gpurun_out/racecheck_final_excl.txt 2>&1; echo rc=$?
grep -E "RACECHECK SUMMARY|ERROR SUMMARY" gpurun_out/racecheck_final_excl.txt | tail -3
grep -E "^=========     (Read|Write) Thread" gpurun_out/racecheck_final_excl.txt | sed -E 's/Thread \([0-9,]+\)//; s/\+0x[0-9a-f]+//' | cut -c1-160 | sort | uniq -c | sort -rn | head -10
