#!/bin/bash
# usage: tools/trace_sweep.sh "ENV=val ..." ...  trace build per variant, prints the steady-state tile line
for v in "$@"; do
  env $v DG_TRACE=1 python -m paper_1710_03887_b200.build --force > /dev/null 2>&1 || { echo "build [$v] failed"; continue; }
  echo "[$v]"; python tools/trace_stage.py C4 | tail -2
done
