#!/bin/bash
# ncu captures of the BASELINE-config kernels at the HEAD build (after plain runs exit 0): C4, C3, C5, N = 2, modal p = 2
mkdir -p gpurun_out
cap() { # name kernel-regex bench-args
  local n=$1 k=$2; shift 2
  local CMD="python bench.py $* --steps 2 --warmup 3 --no-cpu-baseline"
  timeout 300 $CMD > gpurun_out/pre_$n.json 2> gpurun_out/pre_$n.err || { echo "plain $n failed"; return; }
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 5 -c 1 -f -o gpurun_out/prof_$n $CMD > gpurun_out/ncu_$n.log 2>&1; echo "ncu $n rc=$?"
  ncu -i gpurun_out/prof_$n.ncu-rep --page source --csv --print-source cuda,sass > /tmp/prof_${n}_source.csv 2>> gpurun_out/src.err
  # summaries on the box (the reports are too large to bring back): counters, per-line tables
  python tools/ncu_summary.py full gpurun_out/prof_$n.ncu-rep gpurun_out/ncu_summary_$n.json $ELEMS > /dev/null 2>> gpurun_out/src.err
  (echo "# $n: shared-memory wavefronts and stall samples per source line (tools/ncu_smem_lines.py, tools/ncu_lines.py), round-2 final build"; python tools/ncu_smem_lines.py /tmp/prof_${n}_source.csv 2>&1 | head -24 | cut -c1-170; echo; echo "# stall samples per source line"; python tools/ncu_lines.py /tmp/prof_${n}_source.csv 28 2>&1 | cut -c1-190) > gpurun_out/ncu_lines_$n.txt
  rm -f gpurun_out/prof_$n.ncu-rep /tmp/prof_${n}_source.csv
}
ELEMS=1473114; cap C4 stage_ws --config C4
ELEMS=662088; cap C3 stage_ws --config C3
ELEMS=384000; cap C5 stage_ho --config C5
ELEMS=1473114; cap C4_N2 stage_ws --config C4 --order 2
ELEMS=1473114; cap C4_modal2 modal_tile --config C4 --scheme modal --order 2
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 5 -c 40 --csv --log-file gpurun_out/launches_C4.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_l4.log 2>&1; echo "ncu launches C4 rc=$?"
