#!/bin/bash
# GPU suite + bench lines of every config on the in-tree build
mkdir -p gpurun_out
rm -f gpurun_out/parity.jsonl; PARITY_LOG=gpurun_out/parity.jsonl timeout 1800 python -m pytest tests -m gpu -q -rf --durations=10 > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; echo "smoke rc=$?"
for c in C4 C3 C2 C5; do
  timeout 400 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "bench $c rc=$?"
  python - <<PY
import json
try:
    d=json.loads(open("gpurun_out/bench_$c.json").read().strip().splitlines()[-1])
    print("$c", d["value"], d["roofline"]["frac"], d.get("clocks"))
except Exception as e: print("$c parse fail", e)
PY
done
