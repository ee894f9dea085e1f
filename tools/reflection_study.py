"""Desk-scale version of the paper's domain study (§3):
the pulse of a benchmark domain is followed to its outer boundary with point sensors recorded
once per RK step on the GPU (dg_sensors_record), and the records are reduced on the GPU
(dg_spectrum) and on the host to the paper's measures:

* decay exponent: least-squares slope of log(peak |p - p0|) on log(r) over sensors at growing
  distance r from the pulse centre -- a spherical acoustic wave decays like 1/r;
* reflection indicator: spectrum (dB) of a sensor `near` the pass-through boundary minus that of
  a reference sensor further in, averaged over a band (P:281 compares spectra sampled 1 and 2 cm
  from the boundary; reading A22);
* percent of atmosphere of the peak deviation at every sensor.

Domains: C3 (horn in a ball, "A-sphere"; sensors on the -x ray from the throat, away from the
horn) and C4 (horn in the truncated box, "Type B"; sensors on the +x ray from the pulse at the
bell mouth), full size, the configs' own pulses, CFL 0.5, LSERK4.

    python tools/reflection_study.py [C3|C4 ...] > gpurun_out/reflection_study.json

A domain may be followed by the scheme and order, e.g. C3:modal:1 -- the paper's own
modal-quadrature scheme at the paper's order p = 1 -- or C4:nodal:1.
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1710_03887_b200 as dg  # noqa: E402
from paper_1710_03887_b200 import analysis  # noqa: E402
from synth import configs  # noqa: E402

# per domain: the ray (unit direction from the pulse centre), distances of the decay sensors,
# the distance from the centre to the outer boundary along the ray, and the band (Hz, with the
# SPEC time scale 2.915e-5 s per scaled unit) of the reflection indicator
DOMAINS = {
    "C3": dict(direction=(-1.0, 0.0, 0.0), radii=(0.08, 0.12, 0.16, 0.20, 0.25), boundary=0.5),
    "C4": dict(direction=(1.0, 0.0, 0.0), radii=(0.08, 0.12, 0.16, 0.20, 0.25), boundary=0.9),
}
TIME_SCALE = 2.915e-5
NEAR, REF = 0.02, 0.10     # near-boundary and reference sensors: distance from the boundary


def run(spec):
    name, _, rest = spec.partition(":")
    scheme, _, order = rest.partition(":")
    cfg = configs.make(name)
    if order:
        cfg.order = int(order)
    d = DOMAINS[name]
    m = cfg.mesh
    centre = np.array(cfg.pulses[0][2], dtype=np.float64)
    ray = np.array(d["direction"])
    radii = list(d["radii"])
    pts = [centre + r * ray for r in radii]
    pts += [centre + (d["boundary"] - NEAR) * ray, centre + (d["boundary"] - REF) * ray]
    s = dg.Solver(cfg.order, m.vxyz, m.etov, m.bc, etoe=m.etoe, etof=m.etof, gamma=cfg.gamma, q_inf=cfg.q_inf,
                  scheme=dg.DG_SCHEME_MODAL if scheme == "modal" else dg.DG_SCHEME_NODAL)
    s.set_state(configs.initial_state(cfg, s.nodes()))
    dt = s.stable_dt(cfg.cfl)
    owner = s.set_sensors(np.array(pts))
    # follow the pulse to the boundary and a little past it (c0 = 1 in scaled units)
    t_end = d["boundary"] + 0.15
    steps = int(np.ceil(t_end / dt))
    s.record_sensors(steps + 1)
    t0 = time.time()
    s.step(dt, steps)
    torch.cuda.synchronize()
    wall = time.time() - t0
    rec = s.sensor_record()                          # (steps, nsens, 6): rho, mx, my, mz, E, p
    p = torch.as_tensor(rec[:, :, 5], device="cuda")  # pressure records stay on the GPU
    dev = (p - cfg.p0).abs().amax(dim=0).cpu().numpy()
    nd = len(radii)
    slope = analysis.decay_exponent(radii, dev[:nd])
    freqs, db, amp = analysis.spectrum(p[:, nd:nd + 2], dt, TIME_SCALE)   # GPU DFT (dg_spectrum)
    db = db.cpu().numpy()
    # the band that carries the pulse: scaled frequencies 0.2-2 x c0 / (2 pi w) (w = pulse width)
    f0 = 1.0 / (2.0 * np.pi * cfg.pulses[0][1]) / TIME_SCALE
    band = (0.2 * f0, 2.0 * f0)
    diff, refl = analysis.reflection_indicator(db[:, 0], db[:, 1], freqs, band)
    return {
        "domain": name, "scheme": scheme or "nodal", "elements": int(m.K), "order": cfg.order, "dt": dt, "steps": steps, "t_end": steps * dt,
        "wall_s": round(wall, 2), "pulse": cfg.pulses[0], "sensor_points": [list(map(float, q)) for q in pts],
        "sensor_elements": [int(o) for o in owner],
        "decay": {"radii": radii, "peak_dev": [float(v) for v in dev[:nd]], "exponent": slope,
                  "expected": -1.0, "note": "spherical spreading, amplitude ~ 1/r (P:201)"},
        "percent_of_atmosphere": [float(v) for v in analysis.percent_of_atmosphere(dev, cfg.p0)],
        "reflection": {"near_boundary_distance": NEAR, "reference_distance": REF, "band_hz": list(band),
                       "mean_db_difference": refl, "spectrum_bins": int(len(freqs)),
                       "peak_dev_near": float(dev[nd]), "peak_dev_ref": float(dev[nd + 1]),
                       "spreading_only_db": float(20 * np.log10((d["boundary"] - REF) / (d["boundary"] - NEAR)))},
    }


def main():
    names = sys.argv[1:] or ["C3", "C4"]
    out = {"study": "desk-scale domain comparison (SURVEY N4)", "time_scale_s": TIME_SCALE,
           "results": [run(n) for n in names]}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
