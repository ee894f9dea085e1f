"""Aggregate ncu source-page stall samples per CUDA source line.

usage: ncu -i rep --page source --csv --print-source cuda,sass > x.csv; python tools/ncu_lines.py x.csv [N]
"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr = None
cur = None
fname = None
samples = defaultdict(int)
stalls = defaultdict(lambda: defaultdict(int))
src = {}
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        si = hdr.index("Warp Stall Sampling (All Samples)")
        scols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
        continue
    if hdr is None or len(r) <= si:
        continue
    if r[0].strip():
        cur = (fname, int(r[0]))
        src[cur] = r[1]
        continue
    try:
        v = int(r[si])
    except ValueError:
        continue
    samples[cur] += v
    for c in scols:
        try:
            stalls[cur][hdr[c]] += int(r[c])
        except ValueError:
            pass
tot = sum(samples.values()) or 1
print("total samples", tot)
for k, v in sorted(samples.items(), key=lambda kv: -kv[1])[:top]:
    st = ", ".join(f"{a[6:]}={b / v * 100:.0f}%" for a, b in sorted(stalls[k].items(), key=lambda kv: -kv[1])[:3])
    print(f"{k[0][:12]}:{k[1]:4d} {v / tot * 100:5.1f}%  {src.get(k, '')[:64]:64s} {st}")
