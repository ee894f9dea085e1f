#!/bin/bash
# Build variants of the warp split and time one C4 stage for each (experiment helper).
for pw in "$@"; do
  DG_WS_PW=$pw python -m paper_1710_03887_b200.build --force > /dev/null 2>&1 || { echo "build $pw failed"; continue; }
  for d in 0 1 2; do
    DG_DEBUG_TIMING=$d timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | \
      python -c "import json,sys; j=json.loads(sys.stdin.read()); print('PW=$pw debug=$d stage_ms', round(j['ms_per_step']/5,3), 'GDOF/s', j['value'])"
  done
done
