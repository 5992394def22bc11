#!/bin/bash
set -u
echo "== group tests"; timeout 900 python -m pytest tests/test_gpu_group.py -x -q 2>&1 | tail -2
timeout 300 python scripts/pair_time.py 16384 up,down,sq_v32 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l); print(d['shape'], 'groups', d['groups_ms'], 'build', d['group_build_ms'], 'Ku', d['K_union_per_group'])
    except Exception: print(l.strip()[:300])
"
