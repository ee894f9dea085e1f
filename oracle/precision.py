"""The oracle's own fp64 noise floor.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The same RHS algorithm (oracle/rhs.py) evaluated in numpy ``longdouble``
(x87 extended: 64-bit significand, eps = 1.08e-19): reference operators rounded from the
same 50-digit mpmath results to extended precision, affine geometry by cofactors in
extended precision (numpy.linalg has no extended-precision det/inv), the state promoted
exactly.  The difference to the fp64 evaluation on the same input is the fp64 rounding
error of the method itself -- the floor below which no fp64 implementation can be compared,
and the calibration of the 1e-11 parity tolerance."""
from __future__ import annotations

import copy

import numpy as np

from .geom import Geometry, element_vertices
from .refelem import reference_element
from .rhs import OracleMesh, rhs


def geometry_longdouble(vxyz, etov) -> Geometry:
    """SURVEY O2 in extended precision: J, inverse Jacobian (cofactors / J), normals, Fscale."""
    V = element_vertices(np.asarray(vxyz, dtype=np.float64), np.asarray(etov)).astype(np.longdouble)
    a, b, c = (V[:, 1] - V[:, 0]) / 2, (V[:, 2] - V[:, 0]) / 2, (V[:, 3] - V[:, 0]) / 2
    # A = [a b c] (columns dx/dr, dx/ds, dx/dt); rows of A^{-1} = (b x c, c x a, a x b) / det
    J = np.einsum("kd,kd->k", a, np.cross(b, c))
    inv = np.stack([np.cross(b, c), np.cross(c, a), np.cross(a, b)], axis=1) / J[:, None, None]
    gr, gs, gt = inv[:, 0, :], inv[:, 1, :], inv[:, 2, :]
    g = np.stack([-gt, -gs, gr + gs + gt, -gr], axis=1)
    gn = np.sqrt(np.einsum("kfd,kfd->kf", g, g))
    n = g / gn[:, :, None]
    volume = 4 * J / 3
    area = 2 * gn * J[:, None]
    return Geometry(J=J, rx=inv, nx=n, sJ=gn * J[:, None], Fscale=gn, volume=volume, area=area,
                    h=3 * volume / area.max(axis=1))


def longdouble_mesh(mesh: OracleMesh) -> OracleMesh:
    m = copy.copy(mesh)
    m.ref = reference_element(mesh.order, np.longdouble)
    m.geo = geometry_longdouble(mesh.vxyz, mesh.etov)
    return m


def rhs_longdouble(mesh: OracleMesh, Q, t: float = 0.0, elems=None):
    """f(Q, t) by the oracle's algorithm in extended precision (shape like rhs.rhs)."""
    return rhs(longdouble_mesh(mesh), np.asarray(Q, dtype=np.float64).astype(np.longdouble), t, elems)
