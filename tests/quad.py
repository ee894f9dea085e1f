"""Independent numerical-integration helpers for the oracle pins (tests only).

Collapsed (Duffy) Gauss-Legendre rules on the reference tetrahedron and
triangle, and a plain fp64 monomial-in-(r,s,t) evaluation of the Lagrange
basis.  These are a *different route* from oracle/refelem.py (which uses
shifted monomials, exact Dirichlet integrals and 50-digit mpmath), so an error
in either shows up as a mismatch.
"""
import numpy as np


def tet_rule(n: int):
    """Points (r, s, t) and weights of a collapsed n^3 Gauss rule on the reference tet."""
    g, w = np.polynomial.legendre.leggauss(n)
    a, b, c = np.meshgrid(g, g, g, indexing="ij")
    wa, wb, wc = np.meshgrid(w, w, w, indexing="ij")
    r = (1 + a) * (1 - b) * (1 - c) / 4 - 1
    s = (1 + b) * (1 - c) / 2 - 1
    t = c
    wt = wa * wb * wc * (1 - b) * (1 - c) ** 2 / 8
    return r.ravel(), s.ravel(), t.ravel(), wt.ravel()


def tri_rule(n: int):
    """Points (u, v) and weights of a collapsed n^2 Gauss rule on {u, v >= -1, u + v <= 0}."""
    g, w = np.polynomial.legendre.leggauss(n)
    a, b = np.meshgrid(g, g, indexing="ij")
    wa, wb = np.meshgrid(w, w, indexing="ij")
    u = (1 + a) * (1 - b) / 2 - 1
    v = b
    return u.ravel(), v.ravel(), (wa * wb * (1 - b) / 2).ravel()


def face_points(f: int, u, v):
    """Reference-tet points of face f from its 2D parameters (ABI face numbering)."""
    one = -np.ones_like(u)
    if f == 0:
        return u, v, one
    if f == 1:
        return u, one, v
    if f == 2:
        return -1 - u - v, u, v
    return one, u, v


def monomials(N: int):
    return [(a, b, c) for a in range(N + 1) for b in range(N + 1 - a) for c in range(N + 1 - a - b)]


def lagrange_eval(N: int, rn, sn, tn, r, s, t, deriv=None):
    """Values (or r/s/t derivatives) of the nodal Lagrange basis at points (r, s, t).

    Returns (npts, Np).  Built from plain monomials r^a s^b t^c in fp64."""
    ex = monomials(N)

    def mono(rr, ss, tt, d):
        cols = []
        for (a, b, c) in ex:
            if d is None:
                cols.append(rr ** a * ss ** b * tt ** c)
            elif d == 0:
                cols.append(a * rr ** max(a - 1, 0) * ss ** b * tt ** c if a else 0 * rr)
            elif d == 1:
                cols.append(b * rr ** a * ss ** max(b - 1, 0) * tt ** c if b else 0 * rr)
            else:
                cols.append(c * rr ** a * ss ** b * tt ** max(c - 1, 0) if c else 0 * rr)
        return np.stack(cols, axis=-1)

    V = mono(rn, sn, tn, None)
    return mono(np.asarray(r, float), np.asarray(s, float), np.asarray(t, float), deriv) @ np.linalg.inv(V)
