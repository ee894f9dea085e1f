#!/bin/bash
# Round-2 first GPU call: GPU tests as they stand, C3 bench line, ncu capture of the N = 3 stage kernel.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"
timeout 300 python bench.py --config C3 --no-cpu-baseline > gpurun_out/bench_C3.json 2> gpurun_out/bench_C3.err; echo "bench C3 rc=$?"
CMD3="python bench.py --config C3 --steps 2 --warmup 3 --no-cpu-baseline"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stage_ws -s 5 -c 1 -o gpurun_out/prof_C3 $CMD3 > gpurun_out/ncu_f3.log 2>&1; echo "ncu full C3 rc=$?"
