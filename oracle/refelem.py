"""Oracle reference tetrahedron: nodes and nodal operators, built in mpmath.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

What it follows
---------------
* PAPER.md P:407-412 (Appendix A, ``eq:Uj``): the solution on an element is a
  degree-N polynomial; the paper expands it in an L2-orthonormal basis so the
  element mass matrix is a multiple of I.  The nodal build
  stores the same polynomial by its values at Np nodes.  Here the polynomial
  space is spanned by *monomials* and every integral is exact (Dirichlet
  simplex integrals), evaluated in 50-digit mpmath and rounded to fp64 only at
  the end -- a route independent of the library's fp64 orthonormal-Jacobi one.
* reference tet T = {r,s,t >= -1, r+s+t <= -1} with vertices
  v1=(-1,-1,-1), v2=(1,-1,-1), v3=(-1,1,-1), v4=(-1,-1,1); faces
  f0: t=-1 (v1 v2 v3), f1: s=-1 (v1 v2 v4), f2: r+s+t=-1 (v2 v3 v4),
  f3: r=-1 (v1 v3 v4).  This numbering is part of the C ABI (include/dg.h).
* Nodes: warp & blend (Warburton 2006) with blend parameter alpha = 0 (the
  alpha-optimised table is not in the container).  Restated here in
  a symmetric edge form: every edge (A,B) of the regular tetrahedron of side 2
  moves a point by  4 lam_A lam_B w(lam_B - lam_A) (V_B - V_A)/2, where
  w(r) = sum_i (x_i^GLL - x_i^eq) l_i^eq(r) / (1 - r^2) is the 1D
  equispaced-to-Gauss-Lobatto displacement divided by the edge bubble; a
  face warps its interior by the sum over its three edges, blended into the
  volume by  lam_b lam_c lam_d / prod(lam_x + lam_a/2)  (lam_a = barycentric of
  the opposite vertex).  Points on tet edges take the 1D GLL displacement.
* Node order: equispaced lattice index (i, j, k) -- k (t) outermost, then j
  (s), then i (r) innermost -- with i + j + k <= N (ABI convention).
* Dr = V_r V^{-1};  M_ij = int_T l_i l_j;  E[:, f-block] = int_{face f} l_i l_{Fmask_f[j]}
  in the face's 2D parameter measure (area 2, so that Fscale = sJ/J);
  LIFT = M^{-1} E  (Np x 4 Nfp).
"""
from __future__ import annotations

import functools
from dataclasses import dataclass

import mpmath as mp
import numpy as np

DPS = 50

# local vertex indices (0-based) of each face, ABI numbering
FACE_VERTS = ((0, 1, 2), (0, 1, 3), (1, 2, 3), (0, 2, 3))


def n_nodes(N: int) -> int:
    """Np = (N+1)(N+2)(N+3)/6 (BASELINE.json north_star)."""
    return (N + 1) * (N + 2) * (N + 3) // 6


def n_face_nodes(N: int) -> int:
    """Nfp = (N+1)(N+2)/2."""
    return (N + 1) * (N + 2) // 2


def lattice(N: int):
    """Equispaced lattice indices (i, j, k), ABI node order (k outer, i inner)."""
    out = []
    for k in range(N + 1):
        for j in range(N + 1 - k):
            for i in range(N + 1 - k - j):
                out.append((i, j, k))
    return out


def face_mask(N: int) -> np.ndarray:
    """Fmask[f] = ascending node indices on face f, decided on the integer lattice."""
    lat = lattice(N)
    tests = (
        lambda i, j, k: k == 0,            # f0: t = -1
        lambda i, j, k: j == 0,            # f1: s = -1
        lambda i, j, k: i + j + k == N,    # f2: r + s + t = -1
        lambda i, j, k: i == 0,            # f3: r = -1
    )
    fm = [[n for n, ijk in enumerate(lat) if tst(*ijk)] for tst in tests]
    return np.array(fm, dtype=np.int64)


def _legendre_coeffs(N: int):
    """Coefficients (highest first) of the Legendre polynomial P_N, exact in mpf."""
    # Bonnet recurrence (n+1) P_{n+1} = (2n+1) x P_n - n P_{n-1}, lowest-first lists
    p0, p1 = [mp.mpf(1)], [mp.mpf(0), mp.mpf(1)]
    if N == 0:
        return p0[::-1]
    for n in range(1, N):
        nxt = [mp.mpf(0)] * (n + 2)
        for d, c in enumerate(p1):
            nxt[d + 1] += (2 * n + 1) * c
        for d, c in enumerate(p0):
            nxt[d] -= n * c
        p0, p1 = p1, [c / (n + 1) for c in nxt]
    return p1[::-1]


@functools.lru_cache(maxsize=None)
def gll_points(N: int):
    """Gauss-Lobatto-Legendre points on [-1, 1]: +-1 and the roots of P_N' (ascending, mpf)."""
    with mp.workdps(DPS):
        if N == 1:
            return (mp.mpf(-1), mp.mpf(1))
        c = _legendre_coeffs(N)                         # highest first
        deg = len(c) - 1
        dc = [c[i] * (deg - i) for i in range(deg)]     # derivative, highest first
        roots = mp.polyroots(dc, maxsteps=500, extraprec=4 * DPS)
        interior = sorted(mp.re(x) for x in roots)
        return tuple([mp.mpf(-1)] + interior + [mp.mpf(1)])


def _edge_warp(N: int, r):
    """w(r) = sum_i (x_i^GLL - x_i^eq) l_i^eq(r) / (1 - r^2), as a polynomial.

    Endpoint terms vanish (x^GLL = x^eq = +-1); for an interior i the factor
    (r+1)(r-1) of l_i cancels the bubble, leaving 1/(1 - x_i^eq^2)."""
    gll = gll_points(N)
    eq = [mp.mpf(-1) + mp.mpf(2 * i) / N for i in range(N + 1)]
    w = mp.mpf(0)
    for i in range(1, N):
        term = (gll[i] - eq[i]) / (1 - eq[i] ** 2)
        for j in range(1, N):
            if j != i:
                term *= (r - eq[j]) / (eq[i] - eq[j])
        w += term
    return w


def _regular_tet():
    """A regular tetrahedron of edge length 2 (warp & blend lives on it)."""
    s3, s6 = mp.sqrt(3), mp.sqrt(6)
    return [
        (mp.mpf(-1), -1 / s3, -1 / s6),
        (mp.mpf(1), -1 / s3, -1 / s6),
        (mp.mpf(0), 2 / s3, -1 / s6),
        (mp.mpf(0), mp.mpf(0), 3 / s6),
    ]


@functools.lru_cache(maxsize=None)
def nodes_mp(N: int):
    """Warp & blend (alpha = 0) nodes as mpf barycentrics (lam1..lam4) per node."""
    with mp.workdps(DPS):
        Vt = _regular_tet()
        out = []
        for (i, j, k) in lattice(N):
            lam = [mp.mpf(N - i - j - k) / N, mp.mpf(i) / N, mp.mpf(j) / N, mp.mpf(k) / N]
            X = [sum(lam[v] * Vt[v][d] for v in range(4)) for d in range(3)]
            shift = [mp.mpf(0)] * 3

            def edge_term(a, b):
                amp = 4 * lam[a] * lam[b] * _edge_warp(N, lam[b] - lam[a])
                return [amp * (Vt[b][d] - Vt[a][d]) / 2 for d in range(3)]

            nzero = sum(1 for x in lam if x == 0)
            if nzero >= 3:
                pass                                   # vertex: no displacement
            elif nzero == 2:
                a, b = [v for v in range(4) if lam[v] != 0]
                shift = edge_term(a, b)                # tet edge: 1D GLL warp
            else:
                for f, (b, c, d) in enumerate(FACE_VERTS):
                    a = ({0, 1, 2, 3} - {b, c, d}).pop()
                    num = lam[b] * lam[c] * lam[d]
                    if num == 0:
                        continue
                    den = (lam[b] + lam[a] / 2) * (lam[c] + lam[a] / 2) * (lam[d] + lam[a] / 2)
                    blend = num / den
                    for (p, q) in ((b, c), (c, d), (b, d)):
                        et = edge_term(p, q)
                        for dd in range(3):
                            shift[dd] += blend * et[dd]
            Y = [X[d] + shift[d] for d in range(3)]
            # barycentrics of Y in the regular tet
            A = mp.matrix(4, 4)
            for v in range(4):
                for d in range(3):
                    A[d, v] = Vt[v][d]
                A[3, v] = 1
            lamY = mp.lu_solve(A, mp.matrix([Y[0], Y[1], Y[2], 1]))
            out.append(tuple(lamY[v] for v in range(4)))
        return tuple(out)


def _exponents(N: int):
    return [(a, b, c) for a in range(N + 1) for b in range(N + 1 - a) for c in range(N + 1 - a - b)]


@functools.lru_cache(maxsize=None)
def _fact(n):
    return mp.factorial(n)


def _vol_integral(p, q, w):
    """int_T x^p y^q z^w dr ds dt with x=(1+r)/2 etc.: 8 p! q! w! / (p+q+w+3)!."""
    return 8 * _fact(p) * _fact(q) * _fact(w) / _fact(p + q + w + 3)


def _face_integral(f, p, q, w):
    """int_{face f} x^p y^q z^w in the face's 2D parameter measure (area 2).

    The face is a 2-simplex of three barycentrics; the fourth vanishes on it.
    Each parameterisation (r,s), (r,t), (s,t), (s,t) has |d(param)| = 4 |d(unit simplex)|."""
    zero_var = {0: 2, 1: 1, 2: None, 3: 0}[f]    # f0: z=0, f1: y=0, f2: x=1-y-z, f3: x=0
    e = (p, q, w)
    if zero_var is not None:
        if e[zero_var] != 0:
            return mp.mpf(0)
        rest = [e[v] for v in range(3) if v != zero_var]
        return 4 * _fact(rest[0]) * _fact(rest[1]) / _fact(rest[0] + rest[1] + 2)
    return 4 * _fact(p) * _fact(q) * _fact(w) / _fact(p + q + w + 2)


def _obj(shape):
    return np.empty(shape, dtype=object)


_FIX = 240  # fractional bits of the fixed-point products below (~72 digits)


def _dot(A, B):
    """Exact-to-2^-240 product of mpf matrices via Python big-integer fixed point.

    (Plain object-array dot on mpf values is ~20x slower; this is only a
    speed-up of the same product, the rounding is far below fp64.)"""
    to_int = np.frompyfunc(lambda x: int(mp.nint(mp.ldexp(x, _FIX))), 1, 1)
    P = to_int(A).dot(to_int(B))
    back = np.frompyfunc(lambda n: mp.ldexp(mp.mpf(n), -2 * _FIX), 1, 1)
    return back(P)


def _mp_inv(A):
    n = A.shape[0]
    M = mp.matrix(n, n)
    for i in range(n):
        for j in range(n):
            M[i, j] = A[i, j]
    Mi = mp.inverse(M)
    out = _obj((n, n))
    for i in range(n):
        for j in range(n):
            out[i, j] = Mi[i, j]
    return out


@dataclass(frozen=True)
class RefElem:
    N: int
    Np: int
    Nfp: int
    r: np.ndarray
    s: np.ndarray
    t: np.ndarray
    Dr: np.ndarray
    Ds: np.ndarray
    Dt: np.ndarray
    M: np.ndarray          # reference mass matrix (measure dr ds dt)
    Mface: np.ndarray      # (4, Nfp, Nfp) face mass matrices (face parameter measure)
    LIFT: np.ndarray       # Np x 4 Nfp, columns face-major (f, Fmask_f order)
    Fmask: np.ndarray      # (4, Nfp)


@functools.lru_cache(maxsize=None)
def reference_element(N: int, dtype=np.float64) -> RefElem:
    """All nodal operators at order N, exact to fp64 rounding (see module doc).  dtype =
    np.longdouble rounds the same 50-digit results to x87 extended precision instead (the
    fp64 noise-floor measurement, oracle/precision.py)."""
    if N < 1:
        raise ValueError("order N must be >= 1")
    with mp.workdps(DPS):
        lam = nodes_mp(N)
        Np, Nfp = n_nodes(N), n_face_nodes(N)
        ex = _exponents(N)
        # node coordinates in x=(1+r)/2, y=(1+s)/2, z=(1+t)/2 (= barycentrics 2..4)
        xs = [l[1] for l in lam]
        ys = [l[2] for l in lam]
        zs = [l[3] for l in lam]
        V, Vr, Vs, Vt = _obj((Np, Np)), _obj((Np, Np)), _obj((Np, Np)), _obj((Np, Np))
        zero = mp.mpf(0)
        for n in range(Np):
            x, y, z = xs[n], ys[n], zs[n]
            for m, (a, b, c) in enumerate(ex):
                V[n, m] = x ** a * y ** b * z ** c
                # d/dr = (1/2) d/dx etc.
                Vr[n, m] = (a * x ** (a - 1) * y ** b * z ** c / 2) if a > 0 else zero
                Vs[n, m] = (b * x ** a * y ** (b - 1) * z ** c / 2) if b > 0 else zero
                Vt[n, m] = (c * x ** a * y ** b * z ** (c - 1) / 2) if c > 0 else zero
        C = _mp_inv(V)                         # monomial coefficients of the Lagrange basis
        Dr, Ds, Dt = _dot(Vr, C), _dot(Vs, C), _dot(Vt, C)
        G = _obj((Np, Np))
        for m, (a, b, c) in enumerate(ex):
            for mm, (aa, bb, cc) in enumerate(ex):
                G[m, mm] = _vol_integral(a + aa, b + bb, c + cc)
        M = _dot(C.T, _dot(G, C))                  # M_ij = int l_i l_j
        Ginv = _mp_inv(G)
        Fmask = face_mask(N)
        Lcols = []
        Mface = []
        for f in range(4):
            Gf = _obj((Np, Np))
            for m, (a, b, c) in enumerate(ex):
                for mm, (aa, bb, cc) in enumerate(ex):
                    Gf[m, mm] = _face_integral(f, a + aa, b + bb, c + cc)
            GfCF = _dot(Gf, C[:, Fmask[f]])            # Np x Nfp, monomial side
            Mface.append(_dot(C[:, Fmask[f]].T, GfCF))  # int_f l_Fi l_Fj
            # LIFT_f = M^{-1} E_f with M^{-1} = V G^{-1} V^T and E_f = C^T Gf C_F  =>  V G^{-1} Gf C_F
            Lcols.append(_dot(V, _dot(Ginv, GfCF)))
        LIFT = np.concatenate(Lcols, axis=1)

        if dtype == np.float64:
            def f64(A):
                return np.array([[float(v) for v in row] for row in A], dtype=np.float64)
        else:
            def f64(A):
                return np.array([[np.longdouble(mp.nstr(v, 30)) for v in row] for row in A], dtype=np.longdouble)

        r = np.array([float(2 * l[1] - 1) for l in lam])
        s = np.array([float(2 * l[2] - 1) for l in lam])
        t = np.array([float(2 * l[3] - 1) for l in lam])
        return RefElem(N=N, Np=Np, Nfp=Nfp, r=r, s=s, t=t,
                       Dr=f64(Dr), Ds=f64(Ds), Dt=f64(Dt), M=f64(M),
                       Mface=np.stack([f64(m) for m in Mface]), LIFT=f64(LIFT), Fmask=Fmask)
