#!/bin/bash
# Round-2 fifth session: score kernel W loads evict_normal vs evict_first, alternating on one box.
set -u
export HINM_B200_LIB=scripts/libhinm_b200_exp.so
for i in 1 2 3; do
  HINM_SCORES_STREAM=1 python scripts/scores_l2_ab.py
  python scripts/scores_l2_ab.py
done
