"""Instruction counts per stage kernel in the built library (cuobjdump -sass), optionally vs a
saved listing: python tools/sass_count.py [old_listing.txt]"""
import re
import subprocess
import sys


def counts(text):
    cur, cnt = None, {}
    for line in text.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            cur = m.group(1)
            cnt[cur] = {"n": 0, "DMMA": 0, "DFMA": 0, "LDS": 0, "STS": 0}
            continue
        if cur and re.search(r"/\*[0-9a-f]{4,}\*/", line):
            cnt[cur]["n"] += 1
            for k in ("DMMA", "DFMA", "LDS", "STS"):
                if re.search(r"\b" + k + r"\b|\b" + k + r"\.", line):
                    cnt[cur][k] += 1
    return cnt


new = counts(subprocess.run(["cuobjdump", "-sass", "paper_1710_03887_b200/lib/libdg_b200.so"],
                            capture_output=True, text=True).stdout)
old = counts(open(sys.argv[1]).read()) if len(sys.argv) > 1 else {}
for k in sorted(new):
    if "stage" in k or "modal_warp" in k:
        o = old.get(k)
        print(f"{k[:48]:48s} {new[k]}" + (f"  (was {o})" if o and o != new[k] else ""))
