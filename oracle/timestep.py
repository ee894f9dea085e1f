"""Oracle explicit Runge-Kutta time stepping in 2N-storage form.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

SURVEY §8(c) O5: for s = 1..S:  res <- a_s res + dt f(Q, t + c_s dt);  Q <- Q + b_s res.
res starts at 0; t advances by dt per step.

* LSERK4: Carpenter & Kennedy (1994) five-stage, fourth-order 2N-storage
  scheme mandated by BASELINE.json configs C1-C5 (not in the paper).
  Coefficients from the primary source, pinned by the order conditions in
  tests/test_oracle_timestep.py (P-9) rather than trusted.
* HEUN: the paper's "RK2" (SPEC S:308-316 pins Heun) as the same update
  with a = (0, -1), b = (1, 1/2), c = (0, 1).
"""
from __future__ import annotations

import numpy as np

LSERK4_A = (
    0.0,
    -567301805773.0 / 1357537059087.0,
    -2404267990393.0 / 2016746695238.0,
    -3550918686646.0 / 2091501179385.0,
    -1275806237668.0 / 842570457699.0,
)
LSERK4_B = (
    1432997174477.0 / 9575080441755.0,
    5161836677717.0 / 13612068292357.0,
    1720146321549.0 / 2090206949498.0,
    3134564353537.0 / 4481467310338.0,
    2277821191437.0 / 14882151754819.0,
)
LSERK4_C = (
    0.0,
    1432997174477.0 / 9575080441755.0,
    2526269341429.0 / 6820363962896.0,
    2006345519317.0 / 3224310063776.0,
    2802321613138.0 / 2924317926251.0,
)

HEUN_A = (0.0, -1.0)
HEUN_B = (1.0, 0.5)
HEUN_C = (0.0, 1.0)

SCHEMES = {"lserk4": (LSERK4_A, LSERK4_B, LSERK4_C), "heun": (HEUN_A, HEUN_B, HEUN_C)}


def step(f, Q: np.ndarray, res: np.ndarray, t: float, dt: float, scheme: str = "lserk4"):
    """One time step; returns (Q, res, t + dt).  ``f(Q, t)`` is the RHS."""
    a, b, c = SCHEMES[scheme]
    Q = Q.copy()
    res = res.copy()
    for s in range(len(a)):
        k = f(Q, t + c[s] * dt)
        res = a[s] * res + dt * k
        Q = Q + b[s] * res
    return Q, res, t + dt


def integrate(f, Q: np.ndarray, t: float, dt: float, nsteps: int, scheme: str = "lserk4"):
    res = np.zeros_like(Q)
    for _ in range(nsteps):
        Q, res, t = step(f, Q, res, t, dt, scheme)
    return Q, res, t
