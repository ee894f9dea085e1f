#!/bin/bash
# C3 / C2 variants of the N = 3 kernel
mkdir -p gpurun_out
LIB=paper_1710_03887_b200/lib/libdg_b200.so
cp $LIB /tmp/base_libdg.so
for v in base $(ls variants); do
  if [ "$v" = base ]; then cp /tmp/base_libdg.so $LIB; else cp variants/$v/libdg_b200.so $LIB; fi
  for c in C3 C2; do
  out=$(timeout 300 python bench.py --config $c --no-cpu-baseline 2>/dev/null | tail -1)
  echo "$v $c $(echo $out | python -c 'import json,sys; d=json.load(sys.stdin); print(d["value"], d["roofline"]["frac"])' 2>&1 | tail -1)"
  done
done
cp /tmp/base_libdg.so $LIB
