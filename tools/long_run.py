"""Long-run stability record (SURVEY §7 hard part 8): a BASELINE config stepped
for its full step count at CFL 0.5 with the 10 % pulse and no limiter, the blow-up flag
checked every `check` steps inside dg_rk_step (DG_EBLOWUP names the element), and the state
summarised every `every` steps: min rho, min p, max |u|, max |p - p0| / p0.

    python tools/long_run.py C3 [steps] [every] > gpurun_out/long_run_C3.json

The config may carry a scheme and order, e.g. C4:modal:1 (the paper's scheme at its order) or
C4:nodal:1.
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
from synth import configs  # noqa: E402


def main():
    name, _, rest = sys.argv[1].partition(":")
    scheme, _, order = rest.partition(":")
    cfg = configs.make(name)
    if order:
        cfg.order = int(order)
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else cfg.steps
    every = int(sys.argv[3]) if len(sys.argv) > 3 else max(1, steps // 20)
    check = 10
    m = cfg.mesh
    s = dg.Solver(cfg.order, m.vxyz, m.etov, m.bc, etoe=m.etoe, etof=m.etof, gamma=cfg.gamma, q_inf=cfg.q_inf,
                  check_every=check, scheme=dg.DG_SCHEME_MODAL if scheme == "modal" else dg.DG_SCHEME_NODAL)
    s.set_state(configs.initial_state(cfg, s.nodes()))
    dt = s.stable_dt(cfg.cfl)
    g = cfg.gamma
    rows = []

    def summary(n):
        Q = s.get_state(device=True)
        rho = Q[0]
        u2 = (Q[1] ** 2 + Q[2] ** 2 + Q[3] ** 2) / rho ** 2
        p = (g - 1) * (Q[4] - 0.5 * rho * u2)
        rows.append({"step": n, "t": s.time, "min_rho": float(rho.min()), "min_p": float(p.min()),
                     "max_speed": float(u2.sqrt().max()), "max_dp_rel": float((p - cfg.p0).abs().max() / cfg.p0)})

    summary(0)
    t0 = time.time()
    status = "ok"
    n = 0
    try:
        while n < steps:
            k = min(every, steps - n)
            s.step(dt, k)
            n += k
            summary(n)
        dg.dg_check(s.ctx, s.stream)
    except dg.DGError as e:
        status = str(e)
    torch.cuda.synchronize()
    out = {"config": sys.argv[1], "elements": int(m.K), "order": cfg.order, "steps": n, "dt": dt, "cfl": cfg.cfl,
           "t_end": s.time, "check_every": check, "status": status, "wall_s": round(time.time() - t0, 2),
           "min_p_over_run": min(r["min_p"] for r in rows), "min_rho_over_run": min(r["min_rho"] for r in rows),
           "pulses": cfg.pulses, "samples": rows}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
