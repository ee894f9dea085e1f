"""Oracle of the paper's own spatial scheme: orthonormal modal unknowns with Gauss
quadrature.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

What it follows (Appendix A)
------------------------------------------------
* Weak form ``eq:dgma``: for every test function v of the element space
      int_Omega_j v du/dt + int_{dOmega_j} v F*.n - int_Omega_j grad v . F(u) = 0.
* ``eq:Uj``: u_h = sum_i c_i phi_i with {phi_i} orthonormal, so the mass
  matrix is a multiple of I.  Here phi_i is orthonormal on the reference tet T (measure
  dr ds dt), so the physical mass matrix is J I (affine elements): the basis is built by
  Cholesky-orthonormalising the monomials x^a y^b z^c (x = (1+r)/2, ...) against their
  exact Dirichlet Gram matrix in 50-digit mpmath -- a route independent of the library's
  PKDO/Jacobi basis.  Only the spanned space matters for the results compared (nodal
  values of the solution and of f).
* "volume and surface inner products ... computed using 2p and 2p+1 order accurate
  Gauss quadratures" (reading A23): collapsed-coordinate (Stroud) Gauss-Jacobi product
  rules with n = p+1 points per direction -- exact to degree 2p+1 on the tet and on each
  face triangle; 1D rules from scipy.special.roots_jacobi.
* Numerical flux: LLF with lambda the max over the face's quadrature points
  (lambda_mode 0; per point for lambda_mode 1), boundary ghosts as the nodal oracle
  (wall mirror, pass-through q_inf, inflow), the ambient pressure shift of reading A14
  (still exact: the quadrature integrates the constant-flux terms exactly).
* ``eq:ode``: dc/dt = J^{-1} [ J sum_q w_q sum_a dphi_i/dxi_a(q) (grad xi_a . F)(q)
                                  - sum_f sJ_f sum_q w^f_q phi_i(q) F*_n(q) ].
* Face points (reading A23): each face is integrated at ONE set of physical points --
  the face rule in the face parameterisation of its owner (the element with the smaller
  id) -- from both sides, so the discrete face fluxes cancel exactly (conservation).
  Both traces are the elements' polynomials evaluated at those physical points (shifted
  by the face-centroid difference for periodic pairs) through the inverse affine maps --
  no permutation tables.
* State I/O (reading A23): nodal values at the reference nodes <-> coefficients by
  interpolation, c = V^{-1} u, u = V c.
"""
from __future__ import annotations

import functools

import mpmath as mp
import numpy as np
from scipy.special import roots_jacobi

from . import euler
from .refelem import DPS, _exponents, _vol_integral
from .rhs import BC_INFLOW, BC_PASSTHROUGH, BC_WALL, BlowUp, OracleMesh, ambient_pressure

FACE_VERTS = ((0, 1, 2), (0, 1, 3), (1, 2, 3), (0, 2, 3))


@functools.lru_cache(maxsize=None)
def basis_coeffs(N: int) -> np.ndarray:
    """B (Np x Np): phi_i = sum_m B[m, i] mono_m, orthonormal on T (exact Gram, mpmath)."""
    ex = _exponents(N)
    n = len(ex)
    with mp.workdps(DPS):
        G = mp.matrix(n, n)
        for i, (a, b, c) in enumerate(ex):
            for j, (aa, bb, cc) in enumerate(ex):
                G[i, j] = _vol_integral(a + aa, b + bb, c + cc)
        L = mp.cholesky(G)
        Linv = mp.inverse(L)
        return np.array([[float(Linv[j, i]) for j in range(n)] for i in range(n)])   # L^{-T}


def basis(N: int, r, s, t):
    """phi (P, Np) and its (r,s,t) derivatives at points (r, s, t) (arrays of length P)."""
    r, s, t = (np.asarray(v, dtype=np.float64).ravel() for v in (r, s, t))
    x, y, z = (1 + r) / 2, (1 + s) / 2, (1 + t) / 2
    ex = _exponents(N)
    B = basis_coeffs(N)

    def pw(v, k):
        return v ** k if k > 0 else np.ones_like(v)

    M = np.stack([pw(x, a) * pw(y, b) * pw(z, c) for (a, b, c) in ex], axis=1)
    Mr = np.stack([(a * pw(x, a - 1) * pw(y, b) * pw(z, c) / 2) if a else 0 * x for (a, b, c) in ex], axis=1)
    Ms = np.stack([(b * pw(x, a) * pw(y, b - 1) * pw(z, c) / 2) if b else 0 * x for (a, b, c) in ex], axis=1)
    Mt = np.stack([(c * pw(x, a) * pw(y, b) * pw(z, c - 1) / 2) if c else 0 * x for (a, b, c) in ex], axis=1)
    return M @ B, Mr @ B, Ms @ B, Mt @ B


def gauss_jacobi(n: int, alpha: int):
    x, w = roots_jacobi(n, alpha, 0)          # weight (1 - x)^alpha on [-1, 1]
    return np.asarray(x, dtype=np.float64), np.asarray(w, dtype=np.float64)


@functools.lru_cache(maxsize=None)
def tet_rule(n: int):
    """Collapsed Gauss-Jacobi rule on T, n^3 points, exact to degree 2n-1."""
    a, wa = gauss_jacobi(n, 0)
    b, wb = gauss_jacobi(n, 1)
    c, wc = gauss_jacobi(n, 2)
    A, Bb, C = np.meshgrid(a, b, c, indexing="ij")
    W = np.einsum("i,j,k->ijk", wa, wb, wc) / 8.0
    r = (1 + A) * (1 - Bb) * (1 - C) / 4 - 1
    s = (1 + Bb) * (1 - C) / 2 - 1
    return r.ravel(), s.ravel(), C.ravel().copy(), W.ravel()


@functools.lru_cache(maxsize=None)
def tri_rule(n: int):
    """Collapsed Gauss-Jacobi rule on {u, v >= -1, u + v <= 0} (area 2), n^2 points."""
    a, wa = gauss_jacobi(n, 0)
    b, wb = gauss_jacobi(n, 1)
    A, Bb = np.meshgrid(a, b, indexing="ij")
    u = (1 + A) * (1 - Bb) / 2 - 1
    return u.ravel(), Bb.ravel().copy(), (np.outer(wa, wb) / 2.0).ravel()


def face_points(f: int, u, v):
    """Reference (r, s, t) of face-parameter points (u, v) (parameterisations of SURVEY O2)."""
    u, v = np.asarray(u), np.asarray(v)
    m1 = -np.ones_like(u)
    return {0: (u, v, m1), 1: (u, m1, v), 2: (-1 - u - v, u, v), 3: (m1, u, v)}[f]


class ModalOracle:
    def __init__(self, mesh: OracleMesh):
        self.m = mesh
        p = mesh.order
        self.N = p
        self.Np = mesh.Np
        nq = p + 1
        self.vq = tet_rule(nq)
        self.fq = tri_rule(nq)
        ref = mesh.ref
        self.V = basis(p, ref.r, ref.s, ref.t)[0]           # nodal values of phi: (Np nodes, Np modes)
        self.Vinv = np.linalg.inv(self.V)
        r, s, t, w = self.vq
        self.Pq, self.Pr, self.Ps, self.Pt = basis(p, r, s, t)
        self.wq = w
        u, v, wf = self.fq
        self.wf = wf
        self.Pf = [basis(p, *face_points(f, u, v))[0] for f in range(4)]   # (NQF, Np) per face
        self._ft = None

    def to_modal(self, U):
        return np.asarray(U, dtype=np.float64) @ self.Vinv.T

    def to_nodal(self, c):
        return np.asarray(c, dtype=np.float64) @ self.V.T

    def _phys(self, k, r, s, t):
        """Physical coordinates (P, 3) of reference points of element k."""
        v = self.m.vxyz[self.m.etov[k]]
        w = np.stack([-(1 + r + s + t), 1 + r, 1 + s, 1 + t], axis=1) / 2
        return w @ v

    def _basis_at(self, k, x):
        """phi (P, Np) of element k at physical points x (P, 3): (1+r,1+s,1+t) = J^{-1} (x - v1)."""
        rst1 = (x - self.m.vxyz[self.m.etov[k, 0]]) @ self.m.geo.rx[k].T
        return basis(self.N, rst1[:, 0] - 1, rst1[:, 1] - 1, rst1[:, 2] - 1)[0]

    def _face_tables(self):
        """phi of each element (own) and of its neighbour (nbr) at the face's integration
        points, (K, 4, NQF, Np) each; boundary faces: nbr unused (own copy)."""
        if getattr(self, "_ft", None) is None:
            m = self.m
            u, v, wf = self.fq
            verts = m.vxyz[m.etov]
            K = m.K
            own = np.empty((K, 4, len(wf), self.Np))
            nbr = np.empty_like(own)
            for k in range(K):
                for f in range(4):
                    k2, f2 = int(m.etoe[k, f]), int(m.etof[k, f])
                    if m.bc[k, f] != 0 or k <= k2:           # own rule on my face
                        x = self._phys(k, *face_points(f, u, v))
                    else:                                    # the owner's points, shifted onto my face
                        shift = verts[k, list(FACE_VERTS[f])].mean(axis=0) - verts[k2, list(FACE_VERTS[f2])].mean(axis=0)
                        x = self._phys(k2, *face_points(f2, u, v)) + shift
                    own[k, f] = self._basis_at(k, x)
                    if m.bc[k, f] != 0:
                        nbr[k, f] = own[k, f]
                    else:
                        shift = verts[k2, list(FACE_VERTS[f2])].mean(axis=0) - verts[k, list(FACE_VERTS[f])].mean(axis=0)
                        nbr[k, f] = self._basis_at(k2, x + shift)
            self._ft = (own, nbr)
        return self._ft

    def rhs(self, c: np.ndarray, t: float = 0.0) -> np.ndarray:
        m, g, gamma = self.m, self.m.geo, self.m.gamma
        K = m.K
        c = np.asarray(c, dtype=np.float64)
        p_ref = ambient_pressure(m)
        # volume: u at the quadrature points, contravariant fluxes, weak-form integral
        Uq = c @ self.Pq.T                                   # (5, K, NQ)
        rho, uu, vv, ww, pp = euler.primitives(Uq, gamma)
        bad = ~(np.isfinite(Uq).all(axis=0) & (rho > 0) & (pp > 0))
        if np.any(bad):
            raise BlowUp(int(np.argwhere(bad.any(axis=1))[0][0]), t, "rho<=0, p<=0 or non-finite")
        F, G, H = euler.euler_fluxes(Uq, gamma, p_ref)
        out = np.zeros_like(c)
        for a, Pa in enumerate((self.Pr, self.Ps, self.Pt)):
            Ft = (g.rx[:, a, 0][None, :, None] * F + g.rx[:, a, 1][None, :, None] * G
                  + g.rx[:, a, 2][None, :, None] * H)        # (5, K, NQ)
            out += (Ft * self.wq[None, None, :]) @ Pa
        # faces: every face is integrated at one set of physical points, the owner's rule
        # (owner = the element with the smaller id; reading A23), seen from both sides
        own, nbr = self._face_tables()
        tags = np.asarray(m.bc)
        for f in range(4):
            um = np.einsum("ckn,kqn->ckq", c, own[:, f])                         # (5, K, NQF)
            k2 = np.asarray(m.etoe[:, f])
            up = np.einsum("ckn,kqn->ckq", c[:, k2], nbr[:, f])
            n = g.nx[:, f, :].T[:, :, None]                                      # (3, K, 1)
            for tag, ghost in ((BC_WALL, lambda q, nn: euler.ghost_wall(q, nn)),
                               (BC_PASSTHROUGH, lambda q, nn: euler.ghost_passthrough(q, m.q_inf))):
                sel = tags[:, f] == tag
                if np.any(sel):
                    up[:, sel] = ghost(um[:, sel], n[:, sel])
            sel = tags[:, f] == BC_INFLOW
            if np.any(sel):
                qi = euler.inflow_state(t, m.q_inf, gamma, m.inflow_alpha, m.inflow_time_scale,
                                        m.inflow_half_amplitude)
                up[:, sel] = qi[:, None, None]
            lam = euler.llf_lambda(um, up, n, gamma)         # (K, NQF)
            if m.lambda_mode == 0:
                lam = lam.max(axis=1, keepdims=True)
            fstar = euler.llf_flux(um, up, n, gamma, lam, p_ref)   # (5, K, NQF)
            out -= np.einsum("ckq,kq,kqn->ckn", fstar, g.Fscale[:, f][:, None] * self.wf[None, :], own[:, f])
        return out
