#!/bin/bash
# usage: tools/variant_sweep.sh "ENV=val ..." ...   per variant (env applied to build and run): C4 stage
# time (bench) and the steady-state phase trace of CTA 0 (DG_TRACE build); restores the default build
CFG=${SWEEP_CONFIG:-C4}
for v in "$@"; do
  env $v python -m paper_1710_03887_b200.build --force > /dev/null 2>&1 || { echo "build [$v] failed"; continue; }
  env $v timeout 300 python bench.py --config $CFG --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | \
    python -c "import json,sys; j=json.loads(sys.stdin.read()); print('[$v] stage_ms', round(j['ms_per_step']/5,3), 'GDOF/s', j['value'])"
  if [ -z "$NO_TRACE" ]; then
    env $v DG_TRACE=1 python -m paper_1710_03887_b200.build --force > /dev/null 2>&1 || { echo "trace build [$v] failed"; continue; }
    env $v timeout 300 python tools/trace_stage.py $CFG | tail -9
  fi
done
python -m paper_1710_03887_b200.build --force > /dev/null 2>&1
