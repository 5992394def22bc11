#!/bin/bash
set -u
python -m paper_2407_20496_b200.build --experiments --force > /dev/null 2>&1
nvidia-smi --query-gpu=power.draw,clocks.sm --format=csv
timeout 600 python scripts/power_split.py
