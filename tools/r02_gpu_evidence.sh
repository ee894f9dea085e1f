#!/bin/bash
# GPU tests (parity log) + bench C4/C3 + long runs C3 (500 steps) / C4 (1000 steps)
mkdir -p gpurun_out
rm -f gpurun_out/parity.jsonl; PARITY_LOG=gpurun_out/parity.jsonl timeout 1800 python -m pytest tests -m gpu -q -rf --durations=15 > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_C4.json 2> gpurun_out/bench_C4.err; echo "bench C4 rc=$?"
timeout 300 python bench.py --config C3 --no-cpu-baseline > gpurun_out/bench_C3.json 2> gpurun_out/bench_C3.err; echo "bench C3 rc=$?"
timeout 600 python tools/long_run.py C3 500 25 > gpurun_out/long_run_C3.json 2> gpurun_out/long_run_C3.err; echo "long C3 rc=$?"
timeout 900 python tools/long_run.py C4 1000 50 > gpurun_out/long_run_C4.json 2> gpurun_out/long_run_C4.err; echo "long C4 rc=$?"
