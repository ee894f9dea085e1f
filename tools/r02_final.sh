#!/bin/bash
# Round-2 final evidence on one B200 (HEAD build): GPU suite + smoke, every bench line, ncu captures of
# the two low-order kernels (after plain runs of the same commands exited 0).  Outputs under gpurun_out/.
mkdir -p gpurun_out
rm -f gpurun_out/parity.jsonl; PARITY_LOG=gpurun_out/parity.jsonl timeout 2400 python -m pytest tests -m gpu -q -rf --durations=10 > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.txt
timeout 600 python bench.py > gpurun_out/bench_C4.json 2> gpurun_out/bench_C4.err; echo "bench C4 rc=$?"
for c in C5 C3 C2 C1; do timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "bench $c rc=$?"; done
for o in 1 2; do timeout 300 python bench.py --order $o --no-cpu-baseline > gpurun_out/bench_C4_N$o.json 2> gpurun_out/bench_C4_N$o.err; echo "bench N=$o rc=$?"; done
for p in 1 2 3; do timeout 300 python bench.py --scheme modal --order $p --no-cpu-baseline > gpurun_out/bench_modal$p.json 2> gpurun_out/bench_modal$p.err; echo "bench modal p=$p rc=$?"; done
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/bench_*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1]); r=d["roofline"]
        print(f.split("/")[-1], d["value"], r["bound"], r["frac"], "fp64", r.get("fp64_frac"), "hbm", r.get("hbm_frac"), d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
    except Exception as e: print(f, "parse fail", e)
PY
CMD1="python bench.py --order 1 --steps 2 --warmup 3 --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 5 -c 40 --csv --log-file gpurun_out/launches_C4_N1.csv $CMD1 > gpurun_out/ncu_l1.log 2>&1; echo "ncu launches N1 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stage_lo4 -s 5 -c 1 -f -o gpurun_out/prof_C4_N1 $CMD1 > gpurun_out/ncu_fN1.log 2>&1; echo "ncu full N1 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:modal_lo4 -s 5 -c 1 -f -o gpurun_out/prof_C4_modal1 python bench.py --scheme modal --order 1 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_fm1.log 2>&1; echo "ncu full modal1 rc=$?"
for n in C4_N1 C4_modal1; do
  ncu -i gpurun_out/prof_$n.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/prof_${n}_source.csv 2>> gpurun_out/src.err
  ncu -i gpurun_out/prof_$n.ncu-rep --page details > gpurun_out/prof_${n}_details.txt 2>> gpurun_out/src.err
done
echo done
