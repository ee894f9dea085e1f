#!/bin/bash
# ncu --set full capture (with source) of the low-order stage kernel (C4 mesh, order $1), after a plain run exits 0
O=${1:-1}
mkdir -p gpurun_out
CMD="python bench.py --config C4 --order $O --steps 2 --warmup 3 --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/pre_lo$O.json 2> gpurun_out/pre_lo$O.err; echo "plain rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:stage_lo -s 5 -c 1 -f -o gpurun_out/prof_lo$O $CMD > gpurun_out/ncu_lo$O.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/prof_lo$O.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/prof_lo${O}_source.csv 2> gpurun_out/src.err; echo "source rc=$?"
ncu -i gpurun_out/prof_lo$O.ncu-rep --page raw --csv > gpurun_out/prof_lo${O}_raw.csv 2>> gpurun_out/src.err; echo "raw rc=$?"
ncu -i gpurun_out/prof_lo$O.ncu-rep --page details > gpurun_out/prof_lo${O}_details.txt 2>> gpurun_out/src.err; echo "details rc=$?"
