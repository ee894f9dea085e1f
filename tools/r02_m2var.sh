#!/bin/bash
# modal p = 2 variants on the C4 mesh
mkdir -p gpurun_out
LIB=paper_1710_03887_b200/lib/libdg_b200.so
cp $LIB /tmp/base_libdg.so
for v in base $(ls variants); do
  if [ "$v" = base ]; then cp /tmp/base_libdg.so $LIB; else cp variants/$v/libdg_b200.so $LIB; fi
  out=$(timeout 300 python bench.py --config C4 --order 2 --scheme modal --no-cpu-baseline 2>/dev/null | tail -1)
  echo "$v modal p=2 $(echo $out | python -c 'import json,sys; d=json.load(sys.stdin); print(d["value"], d["roofline"]["frac"])' 2>&1 | tail -1)"
done
cp /tmp/base_libdg.so $LIB
