"""Parity metrics and shared helpers for the GPU-vs-oracle tests.

Tolerances (BASELINE.json north_star; reading A14): fields are made
dimensionless by the physical scales S = (rho0, rho0 c0, rho0 c0, rho0 c0, E0)
because a field can be identically ~0 (e.g. rhs_rho at t = 0 of a pulse at rest):

  e_rhs   = max_q |d rhs_q|_inf / S_q  /  max_q |rhs_q|_inf / S_q   <= 1e-11 (one RHS)
  e_state = max_q |d Q_q|_inf / S_q                                 <= 1e-9  (100 RK steps)
"""
import math

import numpy as np

from oracle import euler
from oracle.rhs import OracleMesh

RHS_TOL = 1e-11
STATE_TOL = 1e-9


def scales(cfg):
    c0 = math.sqrt(cfg.gamma * cfg.p0 / cfg.rho0)
    return np.array([cfg.rho0, cfg.rho0 * c0, cfg.rho0 * c0, cfg.rho0 * c0, cfg.p0 / (cfg.gamma - 1.0)])


def e_rhs(gpu, ora, S):
    d = (np.abs(gpu - ora).reshape(5, -1).max(axis=1) / S).max()
    m = (np.abs(ora).reshape(5, -1).max(axis=1) / S).max()
    return d / m


def e_state(gpu, ora, S):
    return (np.abs(gpu - ora).reshape(5, -1).max(axis=1) / S).max()


def e_pert(gpu, ora, q0):
    """The stricter perturbation form of SURVEY §8(c) A14: max_q |dQ_q|_inf / |Q_q - q0_q|_inf
    (fields identically at q0, e.g. the momentum of a pulse at rest at t = 0, are skipped)."""
    q0 = np.asarray(q0, dtype=np.float64).reshape(5, *([1] * (np.ndim(ora) - 1)))
    d = np.abs(gpu - ora).reshape(5, -1).max(axis=1)
    m = np.abs(ora - q0).reshape(5, -1).max(axis=1)
    ok = m > 0
    return float((d[ok] / m[ok]).max())


def record(test, **vals):
    """Append measured parity numbers to $PARITY_LOG (JSON lines) when it is set (GPU evidence
    runs: tools/r02_gpu_tests.sh); a no-op otherwise."""
    import json
    import os
    path = os.environ.get("PARITY_LOG")
    if path:
        with open(path, "a") as f:
            f.write(json.dumps({"test": test, **{k: (float(v) if hasattr(v, "__float__") else v)
                                                 for k, v in vals.items()}}) + "\n")


def oracle_mesh(cfg, lambda_mode=0, **kw):
    m = cfg.mesh
    return OracleMesh(order=cfg.order, vxyz=m.vxyz, etov=m.etov, bc=m.bc, etoe=m.etoe, etof=m.etof,
                      gamma=cfg.gamma, q_inf=cfg.q_inf, lambda_mode=lambda_mode, **kw)


# Stage-kernel grid caps the multi-step tests run under (dg_set_max_ctas): 0 = one CTA per SM
# (the bench launch configuration; on the oracle-sized meshes <= 1 tile per CTA), 2 and 7 = every
# CTA walks many tiles, so the pipelined steady state -- TMA prefetch of the next tiles, input
# refills two tiles ahead, residual tiles arriving a tile early, the partial last tile landing on
# a CTA's j >= 2 -- meets the oracle too.
GRID_CAPS = (0, 2, 7)


def tiles_per_cta(K, order, cap):
    eb = 120 if order == 1 else 16 if order in (3, 4) else 8   # elements per tile
    if order == 2:                       # 48, or 32 on meshes with fewer 48-element tiles than SMs
        eb = 48 if -(-K // 48) >= 148 else 32
    nt = -(-K // eb)
    grid = min(nt, 148) if cap == 0 else min(nt, 148, cap)
    return -(-nt // grid)


def oracle_dt(o: OracleMesh, Q, cfl):
    """CFL rule of DESIGN.md A10 evaluated by the oracle: cfl h_min / ((N+1)^2 max(|u| + c))."""
    rho, u, v, w, p = euler.primitives(Q, o.gamma)
    lam = (np.sqrt(u * u + v * v + w * w) + np.sqrt(o.gamma * p / rho)).max()
    return cfl * o.geo.h.min() / ((o.order + 1) ** 2 * lam)
