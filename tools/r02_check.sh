#!/bin/bash
# GPU suite, then bench lines of every config (no CPU baseline) -- a regression check
mkdir -p gpurun_out
rm -f gpurun_out/parity.jsonl; PARITY_LOG=gpurun_out/parity.jsonl timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/gpu_tests.log
for c in C4 C3 C2 C5; do timeout 300 python bench.py --config $c --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('$c', j['value'], j['roofline']['frac'])"; done
bash tools/r02_modal.sh
