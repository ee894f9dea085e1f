#!/bin/bash
# usage: r02_prof_any.sh NAME KERNEL_REGEX bench-args... : ncu --set full of one launch after a plain run exits 0
NAME=$1; KRE=$2; shift 2
mkdir -p gpurun_out
CMD="python bench.py $* --steps 2 --warmup 3 --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/pre_$NAME.json 2> gpurun_out/pre_$NAME.err; echo "plain rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$KRE -s 5 -c 1 -f -o gpurun_out/prof_$NAME $CMD > gpurun_out/ncu_$NAME.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/prof_$NAME.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/prof_${NAME}_source.csv 2> gpurun_out/src.err; echo "source rc=$?"
ncu -i gpurun_out/prof_$NAME.ncu-rep --page raw --csv > gpurun_out/prof_${NAME}_raw.csv 2>> gpurun_out/src.err; echo "raw rc=$?"
ncu -i gpurun_out/prof_$NAME.ncu-rep --page details > gpurun_out/prof_${NAME}_details.txt 2>> gpurun_out/src.err; echo "details rc=$?"
