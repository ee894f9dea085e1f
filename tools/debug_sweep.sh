#!/bin/bash
# usage: tools/debug_sweep.sh d1 d2 ...   C4 stage time with DG_DEBUG_TIMING=d (timing experiments)
for d in "$@"; do
  DG_DEBUG_TIMING=$d timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | \
    python -c "import json,sys; j=json.loads(sys.stdin.read()); print('debug=$d stage_ms', round(j['ms_per_step']/5,3))"
done
