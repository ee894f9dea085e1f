#!/bin/bash
# usage: r02_modal_var.sh VARIANT: modal GPU tests on the variant, then bench base vs variant at p = 2, 3 (C4 mesh)
V=$1
mkdir -p gpurun_out
LIB=paper_1710_03887_b200/lib/libdg_b200.so
cp $LIB /tmp/base_libdg.so
cp variants/$V/libdg_b200.so $LIB
timeout 1500 python -m pytest tests/test_gpu_modal.py tests/test_gpu_low_order.py -m gpu -x -q -k modal > gpurun_out/gpu_tests_$V.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests_$V.log
for p in 2 3; do
  for v in base $V; do
    if [ "$v" = base ]; then cp /tmp/base_libdg.so $LIB; else cp variants/$v/libdg_b200.so $LIB; fi
    out=$(timeout 300 python bench.py --config C4 --scheme modal --order $p --no-cpu-baseline 2>/dev/null | tail -1)
    echo "$v p=$p $(echo $out | python -c 'import json,sys; d=json.load(sys.stdin); print(d["value"], d["roofline"]["frac"])' 2>&1 | tail -1)"
  done
done
cp /tmp/base_libdg.so $LIB
