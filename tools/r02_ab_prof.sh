#!/bin/bash
# A/B benches of variants/* (no test suite), then an ncu capture of the in-tree build on config $3
mkdir -p gpurun_out
rm -f gpurun_out/variants.jsonl
bash tools/run_variants.sh "${1:-C3 C4}" ${2:-1}
if [ -n "$3" ]; then
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:stage_ws -s 5 -c 1 -o gpurun_out/prof_$3 python bench.py --config $3 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_$3.log 2>&1; echo "ncu $3 rc=$?"
fi
