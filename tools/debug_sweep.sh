#!/bin/bash
# usage (on the GPU box): tools/debug_sweep.sh d1 d2 ...   C4 stage time of builds with
# -DDG_DEBUG_SKIP=d (1 = skip the DMMA contraction, 2 = skip the flux arithmetic; timing
# experiments only -- build them here first: python tools/build_variants.py skip1:DG_DEBUG_SKIP=1 ...)
LIB=paper_1710_03887_b200/lib/libdg_b200.so
cp $LIB /tmp/base_libdg.so
CFG=${CFG:-C4}
for d in "$@"; do
  cp variants/skip$d/libdg_b200.so $LIB
  timeout 300 python bench.py --config $CFG --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | \
    python -c "import json,sys; j=json.loads(sys.stdin.read()); print('$CFG skip=$d stage_ms', round(j['ms_per_step']/5,3))"
done
cp /tmp/base_libdg.so $LIB
