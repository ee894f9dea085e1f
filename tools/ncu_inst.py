"""Per-source-line executed (warp-level) instruction counts from an ncu source csv (cuda,sass)."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
norm = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
hdr = None
cur = None
fname = None
inst = defaultdict(int)
src = {}
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        ii = hdr.index("Instructions Executed")
        continue
    if hdr is None or len(r) <= ii:
        continue
    if r[0].strip():
        cur = (fname, int(r[0]))
        src[cur] = r[1]
        continue
    try:
        inst[cur] += int(r[ii])
    except ValueError:
        pass
tot = sum(inst.values())
print(f"total warp instructions {tot:.3e}  per unit {tot / norm:.1f}")
for k, v in sorted(inst.items(), key=lambda kv: -kv[1])[:int(sys.argv[3]) if len(sys.argv) > 3 else 40]:
    print(f"{k[0][:12]}:{k[1]:4d} {v / norm:9.1f}  {src.get(k, '')[:80]}")
