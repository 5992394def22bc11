#!/bin/bash
set -u
HINM_EXP_FLAGS="" python -m paper_2407_20496_b200.build --experiments --force > /dev/null 2>&1; cp scripts/libhinm_b200_exp.so scripts/lib_v0.so
HINM_EXP_FLAGS="-DHINM_EPI_SLEEP=500" python -m paper_2407_20496_b200.build --experiments --force > /dev/null 2>&1; cp scripts/libhinm_b200_exp.so scripts/lib_v1.so
HINM_EXP_FLAGS="-DHINM_EPI_SLEEP=2000" python -m paper_2407_20496_b200.build --experiments --force > /dev/null 2>&1; cp scripts/libhinm_b200_exp.so scripts/lib_v2.so
timeout 600 python scripts/power_variants.py scripts/lib_v0.so scripts/lib_v1.so scripts/lib_v2.so scripts/lib_v0.so
