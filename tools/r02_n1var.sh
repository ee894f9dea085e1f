#!/bin/bash
# N = 1 variants on the C4 mesh (nodal and modal)
mkdir -p gpurun_out
LIB=paper_1710_03887_b200/lib/libdg_b200.so
cp $LIB /tmp/base_libdg.so
for v in base $(ls variants); do
  if [ "$v" = base ]; then cp /tmp/base_libdg.so $LIB; else cp variants/$v/libdg_b200.so $LIB; fi
  for sch in nodal modal; do
  out=$(timeout 300 python bench.py --config C4 --order 1 --scheme $sch --no-cpu-baseline 2>/dev/null | tail -1)
  echo "$v $sch N=1 $(echo $out | python -c 'import json,sys; d=json.load(sys.stdin); print(d["value"], d["roofline"]["frac"], d["clocks"]["sm_mhz"])' 2>&1 | tail -1)"
  done
done
cp /tmp/base_libdg.so $LIB
