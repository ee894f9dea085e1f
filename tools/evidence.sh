#!/bin/bash
# Round evidence on one B200: bench lines (C4 default, C5), the launch list and one full ncu
# capture of the stage kernel per config.  Outputs under gpurun_out/ (copied to profiles/ by hand).
set -o pipefail
python -m paper_1710_03887_b200.build --force > gpurun_out/build.log 2>&1
python bench.py > gpurun_out/bench_C4.json 2> gpurun_out/bench_C4.err; echo "bench C4 rc=$?"
python bench.py --config C5 --no-cpu-baseline > gpurun_out/bench_C5.json 2> gpurun_out/bench_C5.err; echo "bench C5 rc=$?"
python bench.py --config C3 --no-cpu-baseline > gpurun_out/bench_C3.json 2> gpurun_out/bench_C3.err; echo "bench C3 rc=$?"
python bench.py --config C2 --no-cpu-baseline > gpurun_out/bench_C2.json 2> gpurun_out/bench_C2.err; echo "bench C2 rc=$?"
CMD4="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
CMD5="python bench.py --config C5 --steps 2 --warmup 3 --no-cpu-baseline"
$CMD4 > gpurun_out/plain4.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -s 5 -c 40 --csv --log-file gpurun_out/launches_C4.csv $CMD4 > gpurun_out/ncu_l4.log 2>&1; echo "ncu launches rc=$?"
$CMD4 > gpurun_out/plain4b.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:stage_ws -s 5 -c 1 -o gpurun_out/prof_C4 $CMD4 > gpurun_out/ncu_f4.log 2>&1; echo "ncu full C4 rc=$?"
$CMD5 > gpurun_out/plain5.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:stage_ho -s 5 -c 1 -o gpurun_out/prof_C5 $CMD5 > gpurun_out/ncu_f5.log 2>&1; echo "ncu full C5 rc=$?"
