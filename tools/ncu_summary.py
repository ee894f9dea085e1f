"""Summarise ncu outputs into profiles/ (committed evidence).

usage:
  python tools/ncu_summary.py full  <report.ncu-rep> <out.json> [elements_per_launch]
  python tools/ncu_summary.py launches <launches.csv> <out.txt>
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active": "dmma_pipe_pct",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
    "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active": "shared_pipe_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "launch__registers_per_thread": "registers_per_thread",
    "launch__shared_mem_per_block_dynamic": "dyn_smem_per_block",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed": "smem_wavefront_pct",
    "lts__t_bytes.sum": "l2_bytes",
    "dram__bytes_read.sum.per_second": "dram_read_rate",
    "dram__bytes_write.sum.per_second": "dram_write_rate",
}
SCALE = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0, "ms": 1e-3, "us": 1e-6, "ns": 1e-9, "s": 1.0,
         "Tbyte/s": 1e12, "Gbyte/s": 1e9, "Mbyte/s": 1e6}


def full(rep, out, elems=None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = {"kernel": vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"}
        for k, name in KEYS.items():
            if k in hdr:
                i = hdr.index(k)
                try:
                    v = float(vals[i].replace(",", ""))
                except ValueError:
                    continue
                d[name] = v * SCALE.get(units[i], 1.0)
                d[name + "_unit"] = "s" if units[i] in ("ms", "us", "ns") else ("B" if "byte" in units[i] else units[i])
        if "dram_read" in d and "dram_write" in d:
            d["dram_bytes_per_launch"] = d["dram_read"] + d["dram_write"]
            if elems:
                d["dram_bytes_per_element"] = d["dram_bytes_per_launch"] / elems
        res.append(d)
    summary = res[0] if len(res) == 1 else {"launches": res}
    if len(res) >= 1:
        summary = dict(res[0])
        summary["source"] = rep
        summary["note"] = "one ncu --set full capture (--clock-control none), per launch"
    json.dump(summary, open(out, "w"), indent=1, sort_keys=True)
    print(json.dumps(summary, indent=1, sort_keys=True))


def launches(path, out):
    rows = [r for r in csv.reader(open(path)) if r]
    i0 = [i for i, r in enumerate(rows) if r[0] == "ID"][0]
    hdr, data = rows[i0], rows[i0 + 1:]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = defaultdict(list)
    for r in data:
        agg[r[ki].split("(")[0][:70]].append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in agg.values())
    lines = [f"# ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised launches)",
             f"# {len(data)} launches, total {tot / 1e6:.3f} ms", "kernel | launches | total ms | avg us | share"]
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"{k} | {len(v)} | {sum(v) / 1e6:.3f} | {sum(v) / len(v) / 1e3:.1f} | {sum(v) / tot:.4f}")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    if sys.argv[1] == "full":
        full(sys.argv[2], sys.argv[3], float(sys.argv[4]) if len(sys.argv) > 4 else None)
    else:
        launches(sys.argv[2], sys.argv[3])
