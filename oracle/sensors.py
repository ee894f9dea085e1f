"""Oracle point sensors: locate a point in the mesh and evaluate the nodal solution there.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

What it follows
---------------
* PAPER.md P:220 and Table 2: "the generated pressure was sampled at various
  positions throughout the computational domain" (sensors 1-4 at fixed points);
  SURVEY §8(f) N1.
* Locating: for element k with vertices v1..v4 the affine map
  x = v1 + J (1+r, 1+s, 1+t)^T gives (1+r, 1+s, 1+t) = J^{-1} (x - v1); the point
  is in k when the barycentrics (-(1+r+s+t)/2, (1+r)/2, (1+s)/2, (1+t)/2) are all
  >= -tol.  On shared faces / edges / vertices the smallest element id wins
  (reading A21).
* Evaluation: the solution on an element is the degree-N polynomial with the
  nodal values; its value at (r,s,t) is sum_i Q_i l_i(r,s,t) with the
  Lagrange basis l_i.  Here l_i is built in 50-digit mpmath from the monomial
  basis (l = monomials . V^{-1}, V_nm = monomial m at node n) -- the same
  independent route as oracle/refelem.py, not the library's orthonormal one.
* Pressure at the point (reading A21): from the interpolated conserved
  variables, p = (gamma - 1)(E - |m|^2 / (2 rho))  (Eq. 2).
"""
from __future__ import annotations

import functools

import mpmath as mp
import numpy as np

from . import geom
from .refelem import DPS, _exponents, _mp_inv, n_nodes, nodes_mp


@functools.lru_cache(maxsize=None)
def _lagrange_monomial_coeffs(N: int):
    """C (Np x Np, mpf): l_i(x,y,z) = sum_m C[m, i] x^a y^b z^c with x = (1+r)/2 etc."""
    with mp.workdps(DPS):
        lam = nodes_mp(N)
        ex = _exponents(N)
        Np = n_nodes(N)
        V = np.empty((Np, Np), dtype=object)
        for n in range(Np):
            x, y, z = lam[n][1], lam[n][2], lam[n][3]
            for m, (a, b, c) in enumerate(ex):
                V[n, m] = x ** a * y ** b * z ** c
        return _mp_inv(V)


def interp_weights(N: int, r: float, s: float, t: float) -> np.ndarray:
    """Nodal interpolation weights w_i = l_i(r, s, t), shape (Np,)."""
    C = _lagrange_monomial_coeffs(N)
    with mp.workdps(DPS):
        x, y, z = (1 + mp.mpf(r)) / 2, (1 + mp.mpf(s)) / 2, (1 + mp.mpf(t)) / 2
        mono = [x ** a * y ** b * z ** c for (a, b, c) in _exponents(N)]
        Np = len(mono)
        return np.array([float(mp.fsum(mono[m] * C[m, i] for m in range(Np))) for i in range(Np)])


def locate(vxyz: np.ndarray, etov: np.ndarray, point, tol: float = 1e-10):
    """(k, r, s, t) of the element containing `point` (smallest id on ties), or (-1, nan, nan, nan)."""
    g = geom.geometric_factors(vxyz, etov)
    v1 = np.asarray(vxyz, dtype=np.float64)[np.asarray(etov)[:, 0]]          # (K, 3)
    d = np.asarray(point, dtype=np.float64)[None, :] - v1
    rst1 = np.einsum("kad,kd->ka", g.rx, d)                                   # (1+r, 1+s, 1+t)
    bary = np.concatenate([1.0 - rst1.sum(axis=1, keepdims=True) / 2, rst1 / 2], axis=1)
    inside = np.nonzero(np.all(bary >= -tol, axis=1))[0]
    if len(inside) == 0:
        return -1, np.nan, np.nan, np.nan
    k = int(inside[0])
    r, s, t = rst1[k] - 1.0
    return k, float(r), float(s), float(t)


def sample(N: int, Q: np.ndarray, k: int, r: float, s: float, t: float, gamma: float = 1.4) -> np.ndarray:
    """(rho, m_x, m_y, m_z, E, p) at reference point (r, s, t) of element k; Q is (5, K, Np)."""
    w = interp_weights(N, r, s, t)
    q = Q[:, k, :] @ w
    p = (gamma - 1.0) * (q[4] - 0.5 * (q[1] ** 2 + q[2] ** 2 + q[3] ** 2) / q[0])
    return np.concatenate([q, [p]])
