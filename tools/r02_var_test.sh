#!/bin/bash
# usage: bash tools/r02_var_test.sh VARIANT "CFGS" [pytest -k expr]: GPU suite + bench with variants/VARIANT/libdg_b200.so in place
V=$1; CFGS=${2:-C3}; K=${3:-}
mkdir -p gpurun_out
LIB=paper_1710_03887_b200/lib/libdg_b200.so
cp $LIB /tmp/base_libdg.so
cp variants/$V/libdg_b200.so $LIB
if [ -n "$K" ]; then timeout 1500 python -m pytest tests -m gpu -x -q -k "$K" > gpurun_out/gpu_tests_$V.log 2>&1; else timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_$V.log 2>&1; fi
echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests_$V.log
for c in $CFGS; do
  for v in base $V; do
    if [ "$v" = base ]; then cp /tmp/base_libdg.so $LIB; else cp variants/$v/libdg_b200.so $LIB; fi
    out=$(timeout 300 python bench.py --config $c --no-cpu-baseline 2>/dev/null | tail -1)
    echo "$v $c $(echo $out | python -c 'import json,sys; d=json.load(sys.stdin); print(d["value"], d["roofline"]["frac"])' 2>/dev/null)"
  done
done
cp /tmp/base_libdg.so $LIB
