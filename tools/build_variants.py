"""Build experiment variants of the library side by side (cross-compiled here, no GPU):

    python tools/build_variants.py NAME:KEY=VAL,KEY=VAL NAME2: ...

writes variants/NAME/libdg_b200.so (git-ignored; travels to the GPU box with gpurun).
tools/run_variants.sh copies each over the in-tree library in the box's copy and benches it."""
import os
import sys
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1710_03887_b200 import build as b  # noqa: E402


def one(spec):
    name, _, defs = spec.partition(":")
    d = dict(kv.split("=") for kv in defs.split(",") if kv)
    out = os.path.join(ROOT, "variants", name, "libdg_b200.so")
    b.build(force=True, out=out, extra_defines=d)
    return out


if __name__ == "__main__":
    with ThreadPoolExecutor(4) as ex:
        for o in ex.map(one, sys.argv[1:]):
            print("built", o)
