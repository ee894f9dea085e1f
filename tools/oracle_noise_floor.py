"""fp64 noise floor of the oracle per BASELINE config:
one RHS on a 1k-element sample of the full-size config (the 200 elements with the largest pulse
amplitude + 800 seeded random ones), fp64 vs longdouble (oracle/precision.py), in the parity
metric of tests/parity.py (scaled by S, relative to max |rhs|).  Writes profiles/oracle_noise_floor.json.

    python tools/oracle_noise_floor.py [C1 C2 ...]
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import parity  # noqa: E402
from oracle import geom  # noqa: E402
from oracle.precision import rhs_longdouble  # noqa: E402
from oracle.rhs import rhs  # noqa: E402
from synth import configs  # noqa: E402


def floor(name):
    cfg = configs.make(name)
    o = parity.oracle_mesh(cfg)
    K = cfg.mesh.K
    rng = np.random.default_rng(1)
    cen = cfg.mesh.vxyz[cfg.mesh.etov].mean(axis=1)
    bump = np.zeros(K)
    for amp, w, c in cfg.pulses:
        bump += amp * np.exp(-np.sum((cen - np.asarray(c)) ** 2, axis=1) / w ** 2)
    hot = np.argsort(bump)[-200:]
    sample = np.unique(np.concatenate([hot, rng.choice(K, min(K, 800), replace=False)]))
    patch = np.unique(np.concatenate([sample, cfg.mesh.etoe[sample].ravel()]))
    x = geom.node_coordinates(cfg.mesh.vxyz, cfg.mesh.etov[patch], o.ref.r, o.ref.s, o.ref.t)
    Q = np.zeros((5, K, o.Np))
    Q[:, patch] = configs.initial_state(cfg, x)
    t0 = time.time()
    f64 = rhs(o, Q, 0.0, elems=sample)
    fld = rhs_longdouble(o, Q, 0.0, elems=sample)
    S = parity.scales(cfg)
    d = np.abs(f64 - fld).reshape(5, -1).max(axis=1).astype(np.float64)
    m = np.abs(fld).reshape(5, -1).max(axis=1).astype(np.float64)
    e = float((d / S).max() / (m / S).max())
    return {"config": name, "elements": int(K), "sample": int(len(sample)), "order": cfg.order,
            "e_rhs_fp64_vs_longdouble": e, "per_field_abs": d.tolist(), "max_rhs_abs": m.tolist(),
            "seconds": round(time.time() - t0, 2)}


if __name__ == "__main__":
    names = sys.argv[1:] or ["C1", "C2", "C3", "C4", "C5"]
    out = [floor(n) for n in names]
    for r in out:
        print(r["config"], f"{r['e_rhs_fp64_vs_longdouble']:.2e}")
    path = os.path.join(ROOT, "profiles", "oracle_noise_floor.json")
    json.dump({"what": __doc__.strip().splitlines()[0], "tolerance_rhs": parity.RHS_TOL, "configs": out},
              open(path, "w"), indent=1)
    print("wrote", path)
