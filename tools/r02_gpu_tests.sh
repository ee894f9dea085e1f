#!/bin/bash
# GPU tests + C4/C3 bench lines (round 2 iteration)
mkdir -p gpurun_out
rm -f gpurun_out/parity.jsonl; PARITY_LOG=gpurun_out/parity.jsonl timeout 1800 python -m pytest tests -m gpu -q -rf --durations=15 > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_C4.json 2> gpurun_out/bench_C4.err; echo "bench C4 rc=$?"
timeout 300 python bench.py --config C3 --no-cpu-baseline > gpurun_out/bench_C3.json 2> gpurun_out/bench_C3.err; echo "bench C3 rc=$?"
