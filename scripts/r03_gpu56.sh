#!/bin/bash
set -u
E2E_DIAG=1 timeout 300 python scripts/e2e_sweep.py 2>&1 | tail -1
