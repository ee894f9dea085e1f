#!/bin/bash
# On the GPU box: bench every variants/*/libdg_b200.so (and the in-tree build as "base") on the
# given configs; lines to gpurun_out/variants.jsonl.   usage: bash tools/run_variants.sh "C4 C3" [reps]
CFGS=${1:-C4}; REPS=${2:-1}
mkdir -p gpurun_out
LIB=paper_1710_03887_b200/lib/libdg_b200.so
cp $LIB /tmp/base_libdg.so
for rep in $(seq $REPS); do
for v in base variants/*; do
  name=$(basename $v)
  if [ "$name" = base ]; then cp /tmp/base_libdg.so $LIB; else cp $v/libdg_b200.so $LIB; fi
  for c in $CFGS; do
    out=$(timeout 300 python bench.py --config $c --no-cpu-baseline 2>/dev/null | tail -1)
    echo "{\"variant\": \"$name\", \"config\": \"$c\", \"rep\": $rep, \"line\": $out}" >> gpurun_out/variants.jsonl
    echo "$name $c $(echo $out | python -c 'import json,sys; d=json.load(sys.stdin); print(d["value"], d["roofline"]["frac"])' 2>/dev/null)"
  done
done
done
cp /tmp/base_libdg.so $LIB
