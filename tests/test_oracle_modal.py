"""Pins of the oracle's modal-quadrature scheme (oracle/modal.py; SURVEY §8(f) N3;
PAPER.md Appendix A).

What fixes it, independent of any implementation: the Gauss rules integrate every
monomial of degree <= 2n-1 exactly (Dirichlet integrals); the basis is orthonormal
("multiple of the identity for the mass matrix"); interpolation round-trips; a
uniform state is preserved; the semi-discrete scheme conserves mass, momentum and energy
on a periodic mesh; the exact entropy-wave solution converges at a high-order rate."""
import math

import numpy as np
import pytest

from oracle import modal, timestep
from oracle.refelem import _exponents
from oracle.rhs import OracleMesh
from synth import mesh as smesh

G = 1.4


def _dirichlet3(a, b, c):
    return 8 * math.factorial(a) * math.factorial(b) * math.factorial(c) / math.factorial(a + b + c + 3)


@pytest.mark.parametrize("n", [1, 2, 3, 4])
def test_gauss_rules_exact_to_degree_2n_minus_1(n):
    r, s, t, w = modal.tet_rule(n)
    assert len(w) == n ** 3 and abs(w.sum() - 4.0 / 3.0) < 1e-14
    x, y, z = (1 + r) / 2, (1 + s) / 2, (1 + t) / 2
    for (a, b, c) in _exponents(2 * n - 1):
        exact = _dirichlet3(a, b, c)
        assert abs((w * x ** a * y ** b * z ** c).sum() - exact) < 1e-14 * max(1.0, exact)
    u, v, wf = modal.tri_rule(n)
    assert abs(wf.sum() - 2.0) < 1e-14
    X, Y = (1 + u) / 2, (1 + v) / 2
    for a in range(2 * n):
        for b in range(2 * n - a):
            exact = 4 * math.factorial(a) * math.factorial(b) / math.factorial(a + b + 2)
            assert abs((wf * X ** a * Y ** b).sum() - exact) < 1e-14
    # and not to degree 2n in general (the rule is the stated one, not a finer one)
    a = 2 * n
    assert abs((w * x ** a).sum() - _dirichlet3(a, 0, 0)) > 1e-12


@pytest.mark.parametrize("p", [1, 2, 3])
def test_basis_orthonormal_and_interpolation(p):
    r, s, t, w = modal.tet_rule(p + 1)
    phi = modal.basis(p, r, s, t)[0]
    Gm = (phi * w[:, None]).T @ phi
    assert np.abs(Gm - np.eye(len(Gm))).max() < 1e-13
    o = modal.ModalOracle(OracleMesh(order=p, **_box(3)))
    U = np.random.default_rng(p).normal(size=(5, o.m.K, o.Np))
    assert np.abs(o.to_nodal(o.to_modal(U)) - U).max() < 1e-12
    # derivatives: d/dr of the basis expansion of a polynomial equals the polynomial's derivative
    coef = np.random.default_rng(5).normal(size=o.Np)
    _, pr, ps, pt = modal.basis(p, r, s, t)
    f = lambda rr, ss, tt: (1 + rr) ** p + ss ** p + rr * tt ** (p - 1)  # noqa: E731  (degree p)
    fr = lambda rr, ss, tt: p * (1 + rr) ** (p - 1) + tt ** (p - 1)  # noqa: E731
    cf = np.linalg.lstsq(phi, f(r, s, t), rcond=None)[0]
    assert np.abs(pr @ cf - fr(r, s, t)).max() < 1e-11


def _box(n, periodic=True):
    m = smesh.kuhn_box((n + 1, n, n), (0, 0, 0), (1.3, 1.0, 0.9), periodic=(periodic,) * 3) if periodic else \
        smesh.kuhn_box((n, n, n), (0, 0, 0), (1, 1, 1))
    return dict(vxyz=m.vxyz, etov=m.etov, bc=m.bc, etoe=m.etoe, etof=m.etof, gamma=G)


def _jiggled(n, seed):
    m = smesh.kuhn_box((n, n, n), (0, 0, 0), (1, 1, 1), periodic=(True, True, True))
    rng = np.random.default_rng(seed)
    v = m.vxyz.copy()
    interior = np.all((v > 1e-9) & (v < 1 - 1e-9), axis=1)
    v[interior] += 0.05 / n * rng.uniform(-1, 1, size=(interior.sum(), 3))
    return dict(vxyz=v, etov=m.etov, bc=m.bc, etoe=m.etoe, etof=m.etof, gamma=G)


@pytest.mark.parametrize("p", [1, 2, 3])
def test_free_stream_and_conservation(p):
    o = modal.ModalOracle(OracleMesh(order=p, **_jiggled(3, p)))
    q = np.array([1.2, 0.3, -0.2, 0.1, 2.7])
    U = np.broadcast_to(q[:, None, None], (5, o.m.K, o.Np)).copy()
    f = o.rhs(o.to_modal(U))
    assert np.abs(f).max() < 1e-12
    # conservation: sum_k J_k int_T (sum_i dc_i/dt phi_i) = 0 for every field
    rng = np.random.default_rng(3)
    U = U * (1 + 0.05 * rng.uniform(-1, 1, size=U.shape))
    f = o.rhs(o.to_modal(U))
    r, s, t, w = modal.tet_rule(p + 1)
    mean = (modal.basis(p, r, s, t)[0] * w[:, None]).sum(axis=0)        # int_T phi_i
    tot = np.einsum("k,ckn,n->c", o.m.geo.J, f, mean)
    scale = np.einsum("k,ckn,n->c", o.m.geo.J, np.abs(f), np.abs(mean))
    assert np.all(np.abs(tot) <= 1e-12 * scale), (tot, scale)


@pytest.mark.parametrize("p", [1, 2, 3])
def test_entropy_wave_convergence(p):
    """rho = rho0 (1 + eps sin 2pi(x - u t)), u and p constant: exact Euler solution."""
    vel = np.array([0.3, 0.2, 0.1])
    eps, T = 0.1, 0.1
    errs = []
    for n in (4, 8):
        m = smesh.kuhn_box((n, 3, 3), (0, 0, 0), (1, 3.0 / n, 3.0 / n), periodic=(True, True, True))
        o = modal.ModalOracle(OracleMesh(order=p, vxyz=m.vxyz, etov=m.etov, bc=m.bc, etoe=m.etoe,
                                         etof=m.etof, gamma=G))
        x = o.m.x

        def state(t):
            rho = 1.4 * (1 + eps * np.sin(2 * np.pi * (x[0] - vel[0] * t)))
            E = 1.0 / (G - 1) + 0.5 * rho * (vel @ vel)
            return np.stack([rho, rho * vel[0], rho * vel[1], rho * vel[2], E])

        dt0 = 0.5 * o.m.geo.h.min() / ((p + 1) ** 2 * 1.6)
        nst = int(math.ceil(T / dt0))
        c, _, _ = timestep.integrate(lambda cc, tt: o.rhs(cc, tt), o.to_modal(state(0.0)), 0.0, T / nst, nst)
        e = o.to_nodal(c)[0] - state(T)[0]
        errs.append(math.sqrt(float(np.einsum("k,kn,nm,km->", o.m.geo.J, e, o.m.ref.M, e))))
    rate = math.log(errs[0] / errs[1]) / math.log(2)
    # N + 1/2 is the a-priori bound; coarse meshes run above N + 1 (observed p=1: 3.2)
    assert p + 0.4 <= rate <= p + 2.5, (errs, rate)


@pytest.mark.parametrize("p", [1, 3])
def test_inflow_faces_after_the_pulse_preserve_rest(p):
    """Inflow ghost (Eqs. 5-7) once the pulse is over is the ambient state: rest is preserved;
    during the pulse only elements touching an inflow face feel it (one RHS)."""
    m = smesh.kuhn_box((3, 2, 2), (0, 0, 0), (1, 1, 1), bc_tag=smesh.BC_WALL)
    cen = m.vxyz[m.etov[:, smesh.FACES]].mean(axis=2)
    m.bc[(m.bc != 0) & (cen[:, :, 0] < 1e-9)] = smesh.BC_INFLOW
    o = modal.ModalOracle(OracleMesh(order=p, vxyz=m.vxyz, etov=m.etov, bc=m.bc, etoe=m.etoe, etof=m.etof,
                                     gamma=G, inflow_time_scale=1.0))
    U = np.broadcast_to(np.array([1.4, 0, 0, 0, 2.5])[:, None, None], (5, o.m.K, o.Np)).copy()
    assert np.abs(o.rhs(o.to_modal(U), 2 * np.pi / 565.0 + 1e-6)).max() < 1e-12
    f = o.rhs(o.to_modal(U), np.pi / 565.0)
    touched = (m.bc == smesh.BC_INFLOW).any(axis=1)
    assert np.abs(f[:, touched]).max() > 1e-3 and np.abs(f[:, ~touched]).max() < 1e-12
