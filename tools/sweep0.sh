#!/bin/bash
# usage: tools/sweep0.sh "ENV=val ..." ...   builds each variant and times a C4 stage (debug 0 only)
for v in "$@"; do
  env $v python -m paper_1710_03887_b200.build --force > /dev/null 2>&1 || { echo "build [$v] failed"; continue; }
  timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | \
    python -c "import json,sys; j=json.loads(sys.stdin.read()); print('[$v] stage_ms', round(j['ms_per_step']/5,3), 'GDOF/s', j['value'])"
done
