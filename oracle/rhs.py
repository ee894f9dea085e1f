"""Oracle nodal-DG right-hand side f(Q, t) for the 3D Euler equations.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Follows, step by step, SURVEY §8(c) O4 -- the nodal strong form of the
paper's weak formulation ``eq:dgma`` with the semi-discrete ODE
``eq:ode``:

  1. primitives at every node; rho <= 0, p <= 0 or non-finite -> BlowUp
  2. Euler fluxes F, G, H (Eq. 1, reading A1)
  3. volume:   rhs = - sum_d sum_xi  xi_d (D_xi F_d)     (physical-derivative form)
  4. traces:   q- = Q[vmapM], q+ = Q[vmapP] or a ghost (wall: Eq. 4 / A2;
               pass-through: Eq. 3 / P:154; inflow: Eqs. 5-7, NEXT N1)
  5. lambda_f = max over the face's nodes of max(|u-.n| + c-, |u+.n| + c+)
               (lambda_mode 0) or per node (lambda_mode 1)
  6. F* = 1/2 n.(F(q-) + F(q+)) - 1/2 lambda (q+ - q-)
  7. rhs += LIFT (Fscale * (n.F(q-) - F*))

Fluxes are evaluated with the ambient pressure p_inf = p(q_inf) subtracted from
the momentum rows (reading A14): an exact reformulation (D 1 = 0; n.F(q-) - F*
is invariant under a constant flux shift) that keeps the O(p0) background
pressure out of the cancellations, so the fp64 round-off floor of f stays well
below the 1e-11 parity tolerance at the full BASELINE sizes.

State layout (5, K, Np): field-major, element, node (the public ABI layout).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import conn, euler, geom
from .refelem import reference_element

BC_INTERIOR, BC_WALL, BC_PASSTHROUGH, BC_INFLOW = 0, 1, 2, 3


class BlowUp(RuntimeError):
    def __init__(self, element: int, t: float, what: str):
        super().__init__(f"invalid state ({what}) in element {element} at t={t}")
        self.element = element
        self.t = t


@dataclass
class OracleMesh:
    order: int
    vxyz: np.ndarray
    etov: np.ndarray
    bc: np.ndarray
    gamma: float = 1.4
    q_inf: tuple = (1.4, 0.0, 0.0, 0.0, 2.5)
    etoe: np.ndarray | None = None
    etof: np.ndarray | None = None
    lambda_mode: int = 0
    inflow_alpha: float = 565.0
    inflow_time_scale: float = 2.915e-5      # physical s per scaled time unit (reading A24)
    inflow_half_amplitude: float = 0.05
    _maps: dict = field(default_factory=dict, repr=False)

    def __post_init__(self):
        self.vxyz = np.asarray(self.vxyz, dtype=np.float64)
        self.etov = np.asarray(self.etov, dtype=np.int64)
        self.bc = np.asarray(self.bc, dtype=np.int64)
        self.ref = reference_element(self.order)
        self.K = self.etov.shape[0]
        self.Np = self.ref.Np
        self.Nfp = self.ref.Nfp
        self.geo = geom.geometric_factors(self.vxyz, self.etov)
        if self.etoe is None:
            self.etoe, self.etof = conn.connect_by_hashing(self.etov)
        else:
            self.etoe = np.asarray(self.etoe, dtype=np.int64)
            self.etof = np.asarray(self.etof, dtype=np.int64)
            conn.check_symmetric(self.etoe, self.etof)
        bnd = conn.is_boundary(self.etoe, self.etof)
        if np.any(bnd & (self.bc == BC_INTERIOR)):
            raise ValueError("boundary face without a boundary tag")
        if np.any(~bnd & (self.bc != BC_INTERIOR)):
            raise ValueError("interior face carries a boundary tag")
        self._x = None

    @property
    def x(self):
        """Node coordinates (3, K, Np), computed on first use (large meshes: use vmaps(elems))."""
        if self._x is None:
            self._x = geom.node_coordinates(self.vxyz, self.etov, self.ref.r, self.ref.s, self.ref.t)
        return self._x

    def vmaps(self, elems=None):
        key = None if elems is None else tuple(np.asarray(elems).tolist())
        if key not in self._maps:
            if elems is None or self._x is not None:
                self._maps[key] = conn.build_vmaps(self.x, self.vxyz, self.etov, self.etoe, self.etof,
                                                   self.ref.Fmask, self.geo.h, elems)
            else:
                # sampled use on a large mesh: coordinates of the elements and their neighbours only
                e = np.asarray(elems, dtype=np.int64)
                patch = np.unique(np.concatenate([e, self.etoe[e].ravel()]))
                xs = np.zeros((3, self.K, self.Np))
                xs[:, patch] = geom.node_coordinates(self.vxyz, self.etov[patch], self.ref.r, self.ref.s, self.ref.t)
                self._maps[key] = conn.build_vmaps(xs, self.vxyz, self.etov, self.etoe, self.etof,
                                                   self.ref.Fmask, self.geo.h, e)
        return self._maps[key]


def ambient_pressure(mesh) -> float:
    """p(q_inf), subtracted from the momentum fluxes (reading A14); 0 when q_inf is not a valid
    state (it is then unused: no pass-through or inflow face)."""
    q = np.asarray(mesh.q_inf, dtype=np.float64)
    if not (np.all(np.isfinite(q)) and q[0] > 0):
        return 0.0
    p = float(euler.pressure(q, mesh.gamma))
    return p if np.isfinite(p) and p > 0 else 0.0


def _check_state(mesh: OracleMesh, q: np.ndarray, elems: np.ndarray, t: float):
    rho, u, v, w, p = euler.primitives(q, mesh.gamma)
    bad = ~(np.isfinite(q).all(axis=0) & (rho > 0) & (p > 0))
    if np.any(bad):
        e = int(elems[np.argwhere(bad.any(axis=-1))[0][0]])
        raise BlowUp(e, t, "rho<=0, p<=0 or non-finite")


def rhs(mesh: OracleMesh, Q: np.ndarray, t: float = 0.0, elems=None) -> np.ndarray:
    """f(Q, t) for the elements ``elems`` (default: all), shape (5, E, Np)."""
    ref, g, gamma = mesh.ref, mesh.geo, mesh.gamma
    K, Np, Nfp = mesh.K, mesh.Np, mesh.Nfp
    Q = np.asarray(Q)
    if Q.dtype != np.longdouble:       # longdouble only for the noise floor (oracle/precision.py)
        Q = Q.astype(np.float64, copy=False)
    assert Q.shape == (5, K, Np)
    e = np.arange(K) if elems is None else np.asarray(elems, dtype=np.int64)
    Qe = Q[:, e]
    _check_state(mesh, Qe, e, t)

    p_ref = ambient_pressure(mesh)

    # steps 2-3: volume term
    F, G, H = euler.euler_fluxes(Qe, gamma, p_ref)
    out = np.zeros_like(Qe)
    for a, D in enumerate((ref.Dr, ref.Ds, ref.Dt)):
        for d, Fd in enumerate((F, G, H)):
            out -= g.rx[e, a, d][None, :, None] * (Fd @ D.T)

    # step 4: traces and ghosts
    vmapM, vmapP = mesh.vmaps(None if elems is None else e)
    Qf = Q.reshape(5, K * Np)
    qm = Qf[:, vmapM]                               # (5, E, 4, Nfp)
    qp = Qf[:, vmapP].copy()
    n = np.moveaxis(g.nx[e], 2, 0)[..., None]       # (3, E, 4, 1)
    tag = mesh.bc[e]                                # (E, 4)
    wall = tag == BC_WALL
    if np.any(wall):
        qp[:, wall] = euler.ghost_wall(qm[:, wall], n[:, wall])
    pt = tag == BC_PASSTHROUGH
    if np.any(pt):
        qp[:, pt] = euler.ghost_passthrough(qm[:, pt], mesh.q_inf)
    inf = tag == BC_INFLOW
    if np.any(inf):                                 # NEXT row N1, Eqs. 5-7 (reading A24)
        qi = euler.inflow_state(t, mesh.q_inf, gamma, mesh.inflow_alpha, mesh.inflow_time_scale,
                                mesh.inflow_half_amplitude)
        qp[:, inf] = qi[:, None, None]

    # steps 5-6: LLF flux
    lam = euler.llf_lambda(qm, qp, n, gamma)        # (E, 4, Nfp)
    if mesh.lambda_mode == 0:
        lam = lam.max(axis=2, keepdims=True)
    fm = euler.normal_flux(qm, n, gamma, p_ref)
    fstar = euler.llf_flux(qm, qp, n, gamma, lam, p_ref)

    # step 7: lift
    dF = (fm - fstar) * g.Fscale[e][None, :, :, None]
    out += dF.reshape(5, len(e), 4 * Nfp) @ ref.LIFT.T
    return out
