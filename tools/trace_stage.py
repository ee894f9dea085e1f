"""Phase timeline of one CTA of the C4 stage kernel (needs a DG_TRACE=1 build)."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1710_03887_b200 as dg  # noqa: E402
from synth import configs  # noqa: E402

cfg = configs.make(sys.argv[1] if len(sys.argv) > 1 else "C4")
m = cfg.mesh
s = dg.Solver(cfg.order, m.vxyz, m.etov, m.bc, etoe=m.etoe, etof=m.etof, gamma=cfg.gamma, q_inf=cfg.q_inf)
s.set_state(configs.initial_state(cfg, s.nodes()))
dt = s.stable_dt(0.5)
s.step(dt, 2)
torch.cuda.synchronize()
buf = (C.c_ulonglong * 4096)()
f = dg._lib.dg_debug_trace
f.argtypes = [C.c_void_p, C.POINTER(C.c_ulonglong), C.c_int]
f.restype = C.c_int
assert f(s.ctx, buf, 4096) == 0
all_ = np.array(buf, dtype=np.int64)
t = all_[:1024].reshape(64, 16)
w = all_[1024:1024 + 24 * 16 * 8].reshape(24, 16, 8)
names = {0: "C start", 1: "C XVfull", 2: "C volGEMM", 3: "C XFfull", 4: "C faceGEMM", 5: "C epi", 6: "C eloop", 7: "C barC", 15: "P gathered",
         8: "P start", 9: "P tma", 10: "P XVempty", 11: "P vol", 12: "P fetch", 13: "P XFempty", 14: "P face"}
if cfg.order >= 5:
    names = {0: "start", 1: "inputs", 2: "gathers", 3: "Xfree", 4: "vol", 5: "face", 6: "Xsync", 7: "gemm",
             8: "gsync", 9: "epi"}
t0 = t[2, 0]
for j in range(2, 8):
    row = t[j]
    if cfg.order >= 5:
        print(f"tile {j}: warp0 full-wait {row[10]} loader empty-wait {row[11]}")
    print(f"tile {j}: " + "  ".join(f"{names[e]}={row[e] - t0}" for e in sorted(names, key=lambda e: row[e])))
per = (t[10, 0] - t[2, 0]) / 8
print("cycles per tile (tiles 2..10):", per)
if cfg.order <= 4:
    print("per warp, cycles relative to the consumers' tile start (warp-0 stamp) --")
    print("  consumers: at XV_FULL / passed / GEMMs done / singles reduced / residual ready / epilogue done / IO done")
    print("  producers: at XV_EMPTY / passed / volume done / at XF_EMPTY / passed / face done")
    for j in range(3, 7):
        base = t[j, 0]
        print(f"tile {j}:")
        for k in range(16):
            r = w[j, k] - base
            if (k >= 12) if cfg.order == 3 else (k < 8):   # consumer warps (high ids at N = 3)
                print(f"  C w{k:2d}: {r[4]:6d} {r[5]:6d} {r[0]:6d} {r[2]:6d} {r[3]:6d} {r[1]:6d} {r[6]:6d}")
            else:
                print(f"  P w{k:2d}: {r[4]:6d} {r[5]:6d} {r[0]:6d} {r[6]:6d} {r[7]:6d} {r[1]:6d}")
