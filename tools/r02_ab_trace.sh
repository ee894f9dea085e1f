#!/bin/bash
# GPU parity suite, trace of C4 (trace_lib/), A/B benches of variants/*
mkdir -p gpurun_out
rm -f gpurun_out/parity.jsonl; PARITY_LOG=gpurun_out/parity.jsonl timeout 1200 python -m pytest tests -m gpu -x -q -rf > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests.log
LIB=paper_1710_03887_b200/lib/libdg_b200.so
cp $LIB /tmp/base_lib.so; cp trace_lib/libdg_b200.so $LIB
timeout 300 python tools/trace_stage.py C4 > gpurun_out/trace_C4.txt 2>&1; echo "trace rc=$?"
cp /tmp/base_lib.so $LIB
rm -f gpurun_out/variants.jsonl
bash tools/run_variants.sh "${1:-C4}" ${2:-1}
