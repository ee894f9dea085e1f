#!/bin/bash
# parity of the N = 3, 4 phased-kernel variant on small meshes, then A/B benches
LIB=paper_1710_03887_b200/lib/libdg_b200.so
cp $LIB /tmp/base_lib.so; cp variants/ho34/libdg_b200.so $LIB
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "C3 or C4 or C2" 2>&1 | tail -2
cp /tmp/base_lib.so $LIB
rm -f gpurun_out/variants.jsonl
bash tools/run_variants.sh "C3 C4 C2" 1
