#!/bin/bash
# Round-2 fifth session: score kernel software-pipelined loads / 64-thread CTAs vs the product's.
set -u
export HINM_B200_LIB=scripts/libhinm_b200_exp.so
for i in 1 2; do
  python scripts/scores_l2_ab.py
  HINM_SCORES_PIPE=128 python scripts/scores_l2_ab.py
  HINM_SCORES_PIPE=64 python scripts/scores_l2_ab.py
  HINM_SCORES_NT64=1 python scripts/scores_l2_ab.py
done
