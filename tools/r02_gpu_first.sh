#!/bin/bash
# Round-2 session-2 first GPU call: GPU suite, C4/C3 bench lines, full ncu capture of the N = 3 stage kernel on C3.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
rm -f gpurun_out/parity.jsonl; PARITY_LOG=gpurun_out/parity.jsonl timeout 1200 python -m pytest tests -m gpu -q -rf > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_C4.json 2> gpurun_out/bench_C4.err; echo "bench C4 rc=$?"
timeout 300 python bench.py --config C3 --no-cpu-baseline > gpurun_out/bench_C3.json 2> gpurun_out/bench_C3.err; echo "bench C3 rc=$?"
CMD3="python bench.py --config C3 --steps 2 --warmup 3 --no-cpu-baseline"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stage_ws -s 5 -c 1 -o gpurun_out/prof_C3 $CMD3 > gpurun_out/ncu_f3.log 2>&1; echo "ncu full C3 rc=$?"
