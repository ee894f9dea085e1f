"""Oracle pointwise physics: equation of state, Euler fluxes, ghost states, LLF flux.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

State vector q = (rho, rho u, rho v, rho w, E) as the leading axis.

* pressure: Eq. 2 solved for p:  p = (gamma-1) (E - rho/2 |u|^2)
* fluxes:   Eq. 1, read per SURVEY §8(c) A1: the printed "rho v w + p"
            in the y-flux row 4 and z-flux row 3 is a garble; pressure enters only
            the diagonal momentum entries (the standard Euler flux; SPEC S:280's
            rest-state example F_y = (0,0,1,0,0) agrees).  "E+P" is E+p.
* pass-through ghost: the Eq. 3 ambient state q_inf
* wall ghost: Eq. 4 read per SURVEY A2 as the mirror
            m+ = m- - 2 (m-.n) n, rho+ = rho-, E+ = E- (normal velocity flips sign,
            tangential velocity, rho, p unchanged -- the prose of P:158)
* inflow ghost: Eqs. 5-7 -- NEXT row N1; provided for the pins only.
* LLF flux ("local Lax-Friedrichs Riemann solver"):
            F* = 1/2 n.(F(q-) + F(q+)) - 1/2 lambda (q+ - q-),
            lambda = max(|u-.n| + c-, |u+.n| + c+), c = sqrt(gamma p / rho)
            taken per node here; the per-face max of SURVEY A4 is applied in rhs.py.
"""
from __future__ import annotations

import numpy as np


def primitives(q: np.ndarray, gamma: float):
    rho = q[0]
    u, v, w = q[1] / rho, q[2] / rho, q[3] / rho
    p = (gamma - 1.0) * (q[4] - 0.5 * rho * (u * u + v * v + w * w))
    return rho, u, v, w, p


def pressure(q: np.ndarray, gamma: float = 1.4) -> np.ndarray:
    return primitives(np.asarray(q, dtype=np.float64), gamma)[4]


def euler_fluxes(q: np.ndarray, gamma: float, p_shift: float = 0.0):
    """(F, G, H), each shaped like q: the x, y, z flux vectors of Eq. 1 (reading A1).

    ``p_shift`` subtracts the constant flux (0, p_shift e_d, 0) from the momentum rows
    (reading A14, "background-flux subtraction"): exact for the DG operator,
    which differentiates constants to zero and whose LLF difference n.F(q-) - F* is
    invariant under a constant flux shift; it only removes the O(p0) round-off of the
    ambient pressure."""
    rho, u, v, w, p = primitives(q, gamma)
    E = q[4]
    pm = p - p_shift
    F = np.stack([rho * u, rho * u * u + pm, rho * u * v, rho * u * w, u * (E + p)])
    G = np.stack([rho * v, rho * u * v, rho * v * v + pm, rho * v * w, v * (E + p)])
    H = np.stack([rho * w, rho * u * w, rho * v * w, rho * w * w + pm, w * (E + p)])
    return F, G, H


def normal_flux(q: np.ndarray, n: np.ndarray, gamma: float, p_shift: float = 0.0) -> np.ndarray:
    """n . F(q) with n = (nx, ny, nz) broadcast against q[0]."""
    F, G, H = euler_fluxes(q, gamma, p_shift)
    return n[0] * F + n[1] * G + n[2] * H


def sound_speed(q: np.ndarray, gamma: float) -> np.ndarray:
    rho, _, _, _, p = primitives(q, gamma)
    return np.sqrt(gamma * p / rho)


def ghost_passthrough(qm: np.ndarray, q_inf) -> np.ndarray:
    """Eq. 3 ambient state, whatever the interior."""
    q_inf = np.asarray(q_inf, dtype=np.float64).reshape((5,) + (1,) * (qm.ndim - 1))
    return np.broadcast_to(q_inf, qm.shape).copy()


def ghost_wall(qm: np.ndarray, n: np.ndarray) -> np.ndarray:
    """Mirror of the momentum in the wall plane (Eq. 4, reading A2)."""
    mn = qm[1] * n[0] + qm[2] * n[1] + qm[3] * n[2]
    qp = qm.copy()
    qp[1] = qm[1] - 2.0 * mn * n[0]
    qp[2] = qm[2] - 2.0 * mn * n[1]
    qp[3] = qm[3] - 2.0 * mn * n[2]
    return qp


def inflow_pressure(t, alpha: float = 565.0):
    """p1(t) of P:171-181 (NEXT row N1): 1 + (0.05 - 0.05 cos(alpha t)) for t < 2 pi/alpha."""
    t = np.asarray(t, dtype=np.float64)
    return np.where(t < 2.0 * np.pi / alpha, 1.0 + (0.05 - 0.05 * np.cos(alpha * t)), 1.0)


def ghost_inflow(p_hat, gamma: float = 1.4, p0: float = 1.0, rho0: float = 1.4, c: float = 1.0):
    """Eq. 7: rho = gamma p^(1/gamma) (Eq. 6, C = gamma), u = (p - p0)/(rho0 c) (Eq. 5)."""
    p_hat = np.asarray(p_hat, dtype=np.float64)
    rho = gamma * p_hat ** (1.0 / gamma)
    u = (p_hat - p0) / (rho0 * c)
    E = p_hat / (gamma - 1.0) + 0.5 * rho * u * u
    return np.stack([rho, rho * u, np.zeros_like(rho), np.zeros_like(rho), E])


def inflow_state(t, q_inf, gamma: float, alpha: float = 565.0, time_scale: float = 2.915e-5,
                 half_amplitude: float = 0.05) -> np.ndarray:
    """Inflow ghost of Eqs. 5-7 in the units of the ambient state q_inf
    (reading A24), the form the library evaluates:

      p0 = p(q_inf), rho0 = q_inf[0], c0 = sqrt(gamma p0 / rho0)
      p  = p0 (1 + a - a cos(alpha tau t)) while alpha tau t < 2 pi, else p0
      rho = rho0 (p / p0)^(1/gamma)                                           (Eq. 6)
      u = (p - p0) / (rho0 c0), v = w = 0                                     (Eq. 5)
      E = p / (gamma - 1) + rho u^2 / 2                                       (Eq. 7)

    tau = physical seconds per scaled time unit (1 cm / 343 m/s), alpha in rad per
    physical second.  At the paper's constants (q_inf = Eq. 3, a = 0.05, tau = 1) this is
    ghost_inflow(inflow_pressure(t, alpha)) -- the printed Eq. 7 with C = gamma."""
    q_inf = np.asarray(q_inf, dtype=np.float64)
    p0 = float(pressure(q_inf, gamma))
    rho0 = float(q_inf[0])
    c0 = np.sqrt(gamma * p0 / rho0)
    wt = alpha * time_scale * float(t)
    p = p0 * (1.0 + half_amplitude - half_amplitude * np.cos(wt)) if wt < 2.0 * np.pi else p0
    rho = rho0 * (p / p0) ** (1.0 / gamma)
    u = (p - p0) / (rho0 * c0)
    return np.array([rho, rho * u, 0.0, 0.0, p / (gamma - 1.0) + 0.5 * rho * u * u])


def llf_lambda(qm: np.ndarray, qp: np.ndarray, n: np.ndarray, gamma: float) -> np.ndarray:
    """Per-node max(|u-.n| + c-, |u+.n| + c+)."""
    def speed(q):
        rho, u, v, w, p = primitives(q, gamma)
        return np.abs(u * n[0] + v * n[1] + w * n[2]) + np.sqrt(gamma * p / rho)
    return np.maximum(speed(qm), speed(qp))


def llf_flux(qm: np.ndarray, qp: np.ndarray, n: np.ndarray, gamma: float, lam=None,
             p_shift: float = 0.0) -> np.ndarray:
    """F* = 1/2 n.(F(q-) + F(q+)) - 1/2 lam (q+ - q-); lam defaults to the per-node value."""
    if lam is None:
        lam = llf_lambda(qm, qp, n, gamma)
    return 0.5 * (normal_flux(qm, n, gamma, p_shift) + normal_flux(qp, n, gamma, p_shift)) - 0.5 * lam * (qp - qm)
