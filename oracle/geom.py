"""Oracle geometry of affine tetrahedra.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Follows SURVEY §8(c) O2 (and SPEC S:61-69 for the worked examples):
  x(r,s,t) = 1/2 [ -(1+r+s+t) v1 + (1+r) v2 + (1+s) v3 + (1+t) v4 ]
  J = det d(x,y,z)/d(r,s,t) > 0, (r_x ... t_z) = inverse Jacobian
  outward normals  f0: -grad t,  f1: -grad s,  f2: grad r + grad s + grad t,  f3: -grad r
  n = g/|g|,  sJ = |g| J (face parameter measure, area 2),  Fscale = sJ / J = |g|
  h_k = 3 V_k / max face area  (V_k = 4 J/3, face area = 2 sJ)
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class Geometry:
    J: np.ndarray        # (K,)
    rx: np.ndarray       # (K, 3, 3): rows (r, s, t), columns (x, y, z): rx[k, a, d] = d(a)/d(x_d)
    nx: np.ndarray       # (K, 4, 3) unit outward normals
    sJ: np.ndarray       # (K, 4)
    Fscale: np.ndarray   # (K, 4)
    volume: np.ndarray   # (K,)
    area: np.ndarray     # (K, 4)
    h: np.ndarray        # (K,)


def element_vertices(vxyz: np.ndarray, etov: np.ndarray) -> np.ndarray:
    return vxyz[etov]                      # (K, 4, 3)


def geometric_factors(vxyz: np.ndarray, etov: np.ndarray) -> Geometry:
    V = element_vertices(np.asarray(vxyz, dtype=np.float64), np.asarray(etov))
    # columns dx/dr, dx/ds, dx/dt
    A = np.stack([(V[:, 1] - V[:, 0]) / 2, (V[:, 2] - V[:, 0]) / 2, (V[:, 3] - V[:, 0]) / 2], axis=2)
    J = np.linalg.det(A)
    if np.any(~(J > 0)):
        bad = int(np.argmax(~(J > 0)))
        raise ValueError(f"element {bad} has non-positive Jacobian {J[bad]}")
    inv = np.linalg.inv(A)                 # rows: grad r, grad s, grad t
    gr, gs, gt = inv[:, 0, :], inv[:, 1, :], inv[:, 2, :]
    g = np.stack([-gt, -gs, gr + gs + gt, -gr], axis=1)   # (K, 4, 3)
    gn = np.linalg.norm(g, axis=2)
    n = g / gn[:, :, None]
    sJ = gn * J[:, None]
    volume = 4.0 * J / 3.0                 # |T| = 4/3
    area = 2.0 * sJ                        # face parameter area = 2
    h = 3.0 * volume / area.max(axis=1)
    return Geometry(J=J, rx=inv, nx=n, sJ=sJ, Fscale=gn, volume=volume, area=area, h=h)


def node_coordinates(vxyz: np.ndarray, etov: np.ndarray, r, s, t) -> np.ndarray:
    """Physical node coordinates (3, K, Np) by the affine map of O2."""
    V = element_vertices(np.asarray(vxyz, dtype=np.float64), np.asarray(etov))
    w = np.stack([-(1 + r + s + t), 1 + r, 1 + s, 1 + t], axis=0) / 2   # (4, Np)
    return np.einsum("vn,kvd->dkn", w, V)


def repair_orientation(vxyz: np.ndarray, etov: np.ndarray, bc: np.ndarray):
    """Negative-volume tets repaired by swapping two vertices; the ABI fixes which
    (include/dg.h: local vertices 2 and 3, i.e. EToV columns 1 and 2).  The swap exchanges the
    vertex sets of faces f1 = (v1 v2 v4) and f3 = (v1 v3 v4) (f0 and f2 keep theirs), so the
    caller's boundary tags, given in the input face numbering, move with them.
    Returns (etov, bc, flipped)."""
    V = element_vertices(np.asarray(vxyz, dtype=np.float64), np.asarray(etov))
    A = np.stack([(V[:, 1] - V[:, 0]) / 2, (V[:, 2] - V[:, 0]) / 2, (V[:, 3] - V[:, 0]) / 2], axis=2)
    flip = np.linalg.det(A) < 0
    etov = np.array(etov, dtype=np.int64, copy=True)
    bc = np.array(bc, copy=True)
    etov[flip, 1], etov[flip, 2] = etov[flip, 2].copy(), etov[flip, 1].copy()
    bc[flip, 1], bc[flip, 3] = bc[flip, 3].copy(), bc[flip, 1].copy()
    return etov, bc, flip
