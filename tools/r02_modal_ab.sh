#!/bin/bash
# modal throughput p = 1, 2, 3 for the in-tree build and each variants/*
LIB=paper_1710_03887_b200/lib/libdg_b200.so
cp $LIB /tmp/base_lib.so
for v in base variants/*; do
  name=$(basename $v)
  if [ "$name" = base ]; then cp /tmp/base_lib.so $LIB; else cp $v/libdg_b200.so $LIB; fi
  for p in 1 2 3; do timeout 300 python bench.py --scheme modal --order $p --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('$name modal p=$p', j['value'], j['roofline']['frac'])"; done
done
cp /tmp/base_lib.so $LIB
