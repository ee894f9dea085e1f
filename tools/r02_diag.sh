#!/bin/bash
# phase timelines (trace_lib/ DG_TRACE build) and one-side-skipped stage times (variants/skip*)
mkdir -p gpurun_out
LIB=paper_1710_03887_b200/lib/libdg_b200.so
cp $LIB /tmp/base_lib.so
cp trace_lib/libdg_b200.so $LIB
for c in C4 C3; do timeout 300 python tools/trace_stage.py $c > gpurun_out/trace_$c.txt 2>&1; echo "trace $c rc=$?"; done
cp /tmp/base_lib.so $LIB
for c in C4 C3; do timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('$c base stage_ms', round(j['ms_per_step']/5,3))"; CFG=$c bash tools/debug_sweep.sh 1 2; done
