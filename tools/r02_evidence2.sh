#!/bin/bash
# Round-2 evidence on one B200: GPU suite + smoke, bench lines (C4 default with the CPU
# baseline; C5, C3, C2, C1; modal p = 1..3), the C4 launch list and one full ncu capture per
# kernel family.  Outputs under gpurun_out/ (summaries copied to profiles/ afterwards).
mkdir -p gpurun_out
rm -f gpurun_out/parity.jsonl; PARITY_LOG=gpurun_out/parity.jsonl timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_C4.json 2> gpurun_out/bench_C4.err; echo "bench C4 rc=$?"
for c in C5 C3 C2 C1; do timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "bench $c rc=$?"; done
for p in 1 2 3; do timeout 300 python bench.py --scheme modal --order $p --no-cpu-baseline > gpurun_out/bench_modal$p.json 2> gpurun_out/bench_modal$p.err; echo "bench modal p=$p rc=$?"; done
CMD4="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 5 -c 40 --csv --log-file gpurun_out/launches_C4.csv $CMD4 > gpurun_out/ncu_l4.log 2>&1; echo "ncu launches rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stage_ws -s 5 -c 1 -o gpurun_out/prof_C4 $CMD4 > gpurun_out/ncu_f4.log 2>&1; echo "ncu full C4 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stage_ws -s 5 -c 1 -o gpurun_out/prof_C3 python bench.py --config C3 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_f3.log 2>&1; echo "ncu full C3 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stage_ho -s 5 -c 1 -o gpurun_out/prof_C5 python bench.py --config C5 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_f5.log 2>&1; echo "ncu full C5 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:modal_tile -s 3 -c 1 -o gpurun_out/prof_modal2 python bench.py --scheme modal --order 2 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_m2.log 2>&1; echo "ncu full modal2 rc=$?"
