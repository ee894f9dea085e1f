#!/bin/bash
# refresh after the last kernel change: full GPU suite + smoke, modal p = 1 bench + ncu capture
mkdir -p gpurun_out
rm -f gpurun_out/parity.jsonl; PARITY_LOG=gpurun_out/parity.jsonl timeout 2400 python -m pytest tests -m gpu -q -rf --durations=10 > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.txt
timeout 300 python bench.py --scheme modal --order 1 --no-cpu-baseline > gpurun_out/bench_modal1.json 2> gpurun_out/bench_modal1.err; echo "bench modal p=1 rc=$?"
timeout 300 python bench.py --order 1 --no-cpu-baseline > gpurun_out/bench_C4_N1.json 2> gpurun_out/bench_C4_N1.err; echo "bench N=1 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:modal_lo4 -s 5 -c 1 -f -o gpurun_out/prof_C4_modal1 python bench.py --scheme modal --order 1 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_fm1.log 2>&1; echo "ncu full modal1 rc=$?"
ncu -i gpurun_out/prof_C4_modal1.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/prof_C4_modal1_source.csv 2>> gpurun_out/src.err
python - <<'PY'
import json
for f in ("gpurun_out/bench_modal1.json","gpurun_out/bench_C4_N1.json"):
    d=json.loads(open(f).read().strip().splitlines()[-1]); r=d["roofline"]
    print(f, d["value"], r["bound"], r["frac"], d["clocks"])
PY
