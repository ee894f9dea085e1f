#!/bin/bash
# low orders (the paper's p = 1, 2) on the C4 mesh: nodal N = 1, 2 and modal p = 1, 2, 3; C4 / C3 sanity
mkdir -p gpurun_out
for spec in "C4 0 nodal" "C3 0 nodal" "C4 1 nodal" "C4 2 nodal" "C4 1 modal" "C4 2 modal" "C4 3 modal"; do
  set -- $spec
  extra=""; [ "$2" != 0 ] && extra="--order $2"
  out=$(timeout 400 python bench.py --config $1 $extra --scheme $3 --no-cpu-baseline 2>gpurun_out/low_err.txt | tail -1)
  echo "$out" > gpurun_out/low_$1_$2_$3.json
  echo "$spec $(echo $out | python -c 'import json,sys; d=json.load(sys.stdin); r=d["roofline"]; print(d["value"], r["frac"], r.get("hbm_frac"), d["ms_per_step"])' 2>&1 | tail -1)"
done
