#!/bin/bash
# GPU suite on the in-tree build, then A/B benches of variants/* on the given configs
mkdir -p gpurun_out
rm -f gpurun_out/parity.jsonl; PARITY_LOG=gpurun_out/parity.jsonl timeout 1200 python -m pytest tests -m gpu -x -q -rf > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests.log
rm -f gpurun_out/variants.jsonl
bash tools/run_variants.sh "${1:-C3 C4}" ${2:-1}
