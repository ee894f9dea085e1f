"""Write tests/golden/c2_lserk4_100.npz: the CPU oracle's state after 100 LSERK4 steps of the
full-size C2 config (BASELINE.json configs[1]: 24,576 tets, N = 3, pass-through, 0.5 % pulse).

Calls only oracle/ (and the synth/ input generators); nothing comes from the CUDA path.  The
ODE is eq:ode, stepped by LSERK4 (reading A9) with a
fixed dt from the A10 CFL rule (CFL 0.5) evaluated by the oracle at t = 0.

Stored (the full state is 19.7 MB, so a sample plus full-field properties):
  dt, nsteps, t_end          the run
  elems, Q_elems             the final state of 512 elements: the 256 where the final state
                             departs most from the ambient state and 256 seeded random ones
  mass, energy               sum_k J_k w^T rho_k and sum_k J_k w^T E_k of the whole final state
                             (w = M 1, the oracle's mass-matrix row sums)
  dev_max                    max over all nodes of |Q_q - q_inf,q| per field
Run time here: ~11 min (500 oracle RHS evaluations of ~1.3 s).
    python tests/golden/make_c2_100.py
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import timestep  # noqa: E402
from oracle.rhs import OracleMesh, rhs  # noqa: E402
from oracle import euler  # noqa: E402
from synth import configs  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "c2_lserk4_100.npz")
NSTEPS = 100


def main():
    cfg = configs.make("C2")
    m = cfg.mesh
    o = OracleMesh(order=cfg.order, vxyz=m.vxyz, etov=m.etov, bc=m.bc, etoe=m.etoe, etof=m.etof,
                   gamma=cfg.gamma, q_inf=cfg.q_inf)
    Q0 = configs.initial_state(cfg, o.x)
    rho, u, v, w, p = euler.primitives(Q0, o.gamma)
    lam = (np.sqrt(u * u + v * v + w * w) + np.sqrt(o.gamma * p / rho)).max()
    dt = cfg.cfl * o.geo.h.min() / ((o.order + 1) ** 2 * lam)
    t0 = time.time()
    Q, _, t = timestep.integrate(lambda q, tt: rhs(o, q, tt), Q0, 0.0, dt, NSTEPS)
    print(f"{NSTEPS} steps in {time.time() - t0:.0f} s, t = {t}")
    qinf = np.asarray(cfg.q_inf)[:, None, None]
    dev = np.abs(Q - qinf)
    top = np.argsort(dev.max(axis=(0, 2)))[-256:]
    rng = np.random.default_rng(20)
    rest = np.setdiff1d(np.arange(m.K), top)
    elems = np.sort(np.concatenate([top, rng.choice(rest, 256, replace=False)]))
    wts = o.ref.M.sum(axis=1)                       # w = M 1
    J = o.geo.J
    np.savez_compressed(OUT, dt=dt, nsteps=NSTEPS, t_end=t, elems=elems, Q_elems=Q[:, elems],
                        mass=np.sum(J[:, None] * wts[None, :] * Q[0]),
                        energy=np.sum(J[:, None] * wts[None, :] * Q[4]),
                        dev_max=dev.reshape(5, -1).max(axis=1))
    print("wrote", OUT)


if __name__ == "__main__":
    main()
