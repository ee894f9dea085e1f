"""Build libdg_b200.so in-tree for sm_100a (nvcc cross-compiles; no GPU needed).

    python -m paper_1710_03887_b200.build          # or __graft_entry__.build()

Compiles csrc/*.cpp with g++ and csrc/api.cu with nvcc
(-gencode arch=compute_100a,code=sm_100a -lineinfo), links against the NCCL
that ships with torch (site-packages/nvidia/nccl) with an rpath to it.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIBDIR = os.path.join(HERE, "lib")
LIB = os.path.join(LIBDIR, "libdg_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dir() -> str:
    import nvidia  # the pip NCCL torch itself loads
    for p in nvidia.__path__:
        d = os.path.join(p, "nccl")
        if os.path.exists(os.path.join(d, "include", "nccl.h")):
            return d
    raise RuntimeError("nccl.h not found under site-packages/nvidia/nccl")


def _run(cmd):
    print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*"))) + [os.path.join(ROOT, "include", "dg.h")]


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(s) <= t for s in sources())


def defines() -> dict:
    """Compile-time tuning knobs from the environment (DG_WS_PW=...), for experiments."""
    return {k: os.environ[k] for k in ("DG_WS_PW", "DG_WS_CW", "DG_WS_EB", "DG_HO_KC", "DG_HO_SLOTS", "DG_SDF", "DG_TRACE", "DG_KUNROLL", "DG_NEWTON2", "DG_HO_SDF", "DG_WS_IOW", "DG_SKIP_VOL", "DG_XSV4", "DG_FDENSE", "DG_F1", "DG_SBV", "DG_SWSI", "DG_GATHER2", "DG_SRED2", "DG_ECH", "DG_MODAL_TILE", "DG_MI", "DG_MFP", "DG_DEBUG_SKIP", "DG_IODEFER", "DG_CHI") if k in os.environ}


def build(force: bool = False, verbose_ptxas: bool = False, out: str = LIB, extra_defines=None) -> str:
    """Build the library to `out` (default: the in-tree lib/libdg_b200.so the binding loads);
    extra_defines (dict) add compile-time experiment knobs (tools/build_variants.py)."""
    if not force and out == LIB and up_to_date():
        return LIB
    os.makedirs(os.path.dirname(out), exist_ok=True)
    bdir = os.path.join(HERE, "build" if out == LIB else "build_" + os.path.basename(os.path.dirname(out)))
    os.makedirs(bdir, exist_ok=True)
    nd = nccl_dir()
    inc = ["-I", os.path.join(ROOT, "include"), "-I", os.path.join(nd, "include")]
    objs = []
    for src in ("refelem.cpp", "mesh.cpp"):
        o = os.path.join(bdir, src + ".o")
        _run(["g++", "-O2", "-std=c++17", "-fPIC", "-Wall", "-c", os.path.join(CSRC, src), "-o", o] + inc)
        objs.append(o)
    o = os.path.join(bdir, "api.cu.o")
    extra = ["-Xptxas", "-v"] if verbose_ptxas else []
    extra += [f"-D{k}={v}" for k, v in defines().items()]
    extra += [f"-D{k}={v}" for k, v in (extra_defines or {}).items()]
    _run([NVCC] + ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
                          "-c", os.path.join(CSRC, "api.cu"), "-o", o] + inc + extra)
    objs.append(o)
    ncl = os.path.join(nd, "lib")
    _run([NVCC] + ARCH + ["-shared", "-o", out] + objs +
         ["-L", ncl, "-l:libnccl.so.2", "-Xlinker", "-rpath=" + ncl])
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose_ptxas="-v" in sys.argv)
