#!/bin/bash
# traces of C3 and C4 (trace_lib/), then A/B benches of variants/*
mkdir -p gpurun_out
LIB=paper_1710_03887_b200/lib/libdg_b200.so
cp $LIB /tmp/base_lib.so; cp trace_lib/libdg_b200.so $LIB
for c in C4 C3; do timeout 300 python tools/trace_stage.py $c > gpurun_out/trace_$c.txt 2>&1; echo "trace $c rc=$?"; done
cp /tmp/base_lib.so $LIB
rm -f gpurun_out/variants.jsonl
bash tools/run_variants.sh "${1:-C4}" ${2:-1}
