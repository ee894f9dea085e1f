#!/bin/bash
# usage: tools/sweep.sh "ENV=val ENV2=val" ...   builds each variant, times a C4 stage with debug modes 0..3
for v in "$@"; do
  env $v python -m paper_1710_03887_b200.build --force > /dev/null 2>&1 || { echo "build [$v] failed"; continue; }
  for d in 0 1 2 3; do
    DG_DEBUG_TIMING=$d timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | \
      python -c "import json,sys; j=json.loads(sys.stdin.read()); print('[$v] debug=$d stage_ms', round(j['ms_per_step']/5,3), 'GDOF/s', j['value'])"
  done
done
