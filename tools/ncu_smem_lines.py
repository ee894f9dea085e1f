"""Shared-memory wavefronts (actual, ideal, excessive) and stall samples per CUDA source line.

usage: ncu -i rep --page source --csv --print-source cuda,sass > x.csv; python tools/ncu_smem_lines.py x.csv [N]
"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
hdr = None
cur = None
fname = None
agg = defaultdict(lambda: [0, 0, 0, 0])
src = {}
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        iw, ii, ie, ss = (hdr.index("L1 Wavefronts Shared"), hdr.index("L1 Wavefronts Shared Ideal"),
                          hdr.index("L1 Wavefronts Shared Excessive"), hdr.index("Warp Stall Sampling (All Samples)"))
        continue
    if hdr is None or len(r) <= iw:
        continue
    if r[0].strip():
        cur = (fname, int(r[0]))
        src[cur] = r[1]
        continue
    for j, c in enumerate((iw, ii, ie, ss)):
        try:
            agg[cur][j] += int(float(r[c] or 0))
        except ValueError:
            pass
tw = sum(v[0] for v in agg.values()) or 1
ts = sum(v[3] for v in agg.values()) or 1
print(f"total shared wavefronts {tw}, stall samples {ts}")
print("line | wavefronts % | ideal | excessive | samples % | source")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{k[0][:10]}:{k[1]:4d} {v[0] / tw * 100:5.1f}% {v[1]:>10d} {v[2]:>10d} {v[3] / ts * 100:5.1f}%  {src.get(k, '').strip()[:70]}")
