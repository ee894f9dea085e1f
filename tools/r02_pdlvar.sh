#!/bin/bash
mkdir -p gpurun_out
LIB=paper_1710_03887_b200/lib/libdg_b200.so
cp $LIB /tmp/base_libdg.so
for v in base $(ls variants); do
  if [ "$v" = base ]; then cp /tmp/base_libdg.so $LIB; else cp variants/$v/libdg_b200.so $LIB; fi
  for spec in "C4 0" "C2 0" "C1 0" "C4 2"; do set -- $spec; extra=""; [ "$2" != 0 ] && extra="--order $2"
  out=$(timeout 300 python bench.py --config $1 $extra --no-cpu-baseline 2>/dev/null | tail -1)
  echo "$v $1 N$2 $(echo $out | python -c 'import json,sys; d=json.load(sys.stdin); print(d["value"], d["roofline"]["frac"])' 2>&1 | tail -1)"
  done
done
cp /tmp/base_libdg.so $LIB
