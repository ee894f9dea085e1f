#!/bin/bash
# per-warp phase traces of the N = 3 stage kernel (DG_TRACE builds in variants/t*)
mkdir -p gpurun_out
LIB=paper_1710_03887_b200/lib/libdg_b200.so
cp $LIB /tmp/base_libdg.so
for v in variants/t*; do
  n=$(basename $v); cp $v/libdg_b200.so $LIB
  if [[ $n == tpp* ]]; then export TRACE_WARPS=20; else export TRACE_WARPS=16; fi
  timeout 300 python tools/trace_stage.py ${1:-C3} > gpurun_out/trace_$n.txt 2>&1; echo "$n rc=$?"
done
cp /tmp/base_libdg.so $LIB
