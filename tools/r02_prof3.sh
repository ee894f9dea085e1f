#!/bin/bash
# ncu --set full capture (with source) of the N = 3 stage kernel on C3, after a plain run exits 0
mkdir -p gpurun_out
CMD3="python bench.py --config C3 --steps 2 --warmup 3 --no-cpu-baseline"
timeout 300 $CMD3 > gpurun_out/pre_C3.json 2> gpurun_out/pre_C3.err; echo "plain rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:stage_ws -s 5 -c 1 -o gpurun_out/prof_C3 $CMD3 > gpurun_out/ncu_f3.log 2>&1; echo "ncu full C3 rc=$?"
ncu -i gpurun_out/prof_C3.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/prof_C3_source.csv 2> gpurun_out/src.err; echo "source rc=$?"
ncu -i gpurun_out/prof_C3.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_C3_sass.csv 2>> gpurun_out/src.err; echo "sass rc=$?"
ncu -i gpurun_out/prof_C3.ncu-rep --page raw --csv > gpurun_out/prof_C3_raw.csv 2>> gpurun_out/src.err; echo "raw rc=$?"
ls -la gpurun_out/ | head -30
