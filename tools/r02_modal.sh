#!/bin/bash
# modal-scheme throughput p = 1, 2, 3 (C4 mesh)
for p in 1 2 3; do timeout 300 python bench.py --scheme modal --order $p --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('modal p=$p', j['value'], j['unit'], j['roofline']['frac'])"; done
