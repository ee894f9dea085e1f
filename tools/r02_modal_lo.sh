#!/bin/bash
# modal p = 1 four-lane kernel: modal GPU tests + bench on the C4 mesh
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_modal.py -m gpu -x -q > gpurun_out/gpu_tests_modal.log 2>&1; echo "tests rc=$?"; tail -12 gpurun_out/gpu_tests_modal.log
for o in 1; do
  out=$(timeout 400 python bench.py --config C4 --order $o --scheme modal --no-cpu-baseline 2>gpurun_out/modal_err_$o.txt | tail -1)
  echo "$out" > gpurun_out/modal_C4_$o.json
  echo "p=$o $(echo $out | python -c 'import json,sys; d=json.load(sys.stdin); r=d["roofline"]; print(d["value"], r["frac"], r.get("hbm_frac"), d["ms_per_step"])' 2>&1 | tail -1)"
done
