#!/bin/bash
# low-order kernel: GPU suite + N = 1, 2 bench on the C4 mesh
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q ${1:+-k "$1"} > gpurun_out/gpu_tests_lo.log 2>&1; echo "tests rc=$?"; tail -15 gpurun_out/gpu_tests_lo.log
for o in 1 2; do
  out=$(timeout 400 python bench.py --config C4 --order $o --no-cpu-baseline 2>gpurun_out/lo_err_$o.txt | tail -1)
  echo "$out" > gpurun_out/lo_C4_$o.json
  echo "N=$o $(echo $out | python -c 'import json,sys; d=json.load(sys.stdin); r=d["roofline"]; print(d["value"], r["frac"], r.get("hbm_frac"), d["ms_per_step"])' 2>&1 | tail -1)"
done
