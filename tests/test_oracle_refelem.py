"""Pins of the oracle's reference element.

Each check is fixed by the mathematics, not by re-running the oracle's own
formulas: textbook GLL points, the equispaced lattice for N <= 2, exact
differentiation of polynomials written in (r, s, t) (the oracle works in
shifted monomials, so a dropped chain-rule factor fails here), volume/face
integrals by an independent collapsed Gauss rule, and summation by parts.
"""
import itertools
import math

import numpy as np
import pytest

from oracle import refelem
import quad

ORDERS = [1, 2, 3, 4, 5, 6]


@pytest.fixture(scope="module", params=ORDERS)
def R(request):
    return refelem.reference_element(request.param)


def test_counts(R):
    N = R.N
    assert R.Np == (N + 1) * (N + 2) * (N + 3) // 6
    assert R.Fmask.shape == (4, (N + 1) * (N + 2) // 2)


def test_gll_closed_forms():
    g2 = [float(x) for x in refelem.gll_points(2)]
    g3 = [float(x) for x in refelem.gll_points(3)]
    g4 = [float(x) for x in refelem.gll_points(4)]
    assert np.allclose(g2, [-1, 0, 1], atol=1e-15)
    assert np.allclose(g3, [-1, -1 / math.sqrt(5), 1 / math.sqrt(5), 1], atol=1e-15)
    assert np.allclose(g4, [-1, -math.sqrt(3 / 7), 0, math.sqrt(3 / 7), 1], atol=1e-15)


@pytest.mark.parametrize("N", [1, 2])
def test_low_order_nodes_are_equispaced(N):
    R = refelem.reference_element(N)
    lat = np.array(refelem.lattice(N), dtype=float)
    assert np.allclose(R.r, -1 + 2 * lat[:, 0] / N, atol=1e-15)
    assert np.allclose(R.s, -1 + 2 * lat[:, 1] / N, atol=1e-15)
    assert np.allclose(R.t, -1 + 2 * lat[:, 2] / N, atol=1e-15)


def test_edge_nodes_are_gll(R):
    # edge v1-v2 is s = t = -1; its nodes must be the GLL points in r
    on = np.where((np.abs(R.s + 1) < 1e-13) & (np.abs(R.t + 1) < 1e-13))[0]
    g = np.array([float(x) for x in refelem.gll_points(R.N)])
    assert len(on) == R.N + 1
    assert np.allclose(np.sort(R.r[on]), g, atol=1e-14)


def test_nodes_inside_and_on_faces(R):
    lam = np.stack([-(1 + R.r + R.s + R.t) / 2, (1 + R.r) / 2, (1 + R.s) / 2, (1 + R.t) / 2])
    assert lam.min() > -1e-14
    planes = [R.t + 1, R.s + 1, R.r + R.s + R.t + 1, R.r + 1]
    for f in range(4):
        on = np.where(np.abs(planes[f]) < 1e-13)[0]
        assert np.array_equal(on, R.Fmask[f])


def test_face_node_sets_symmetric(R):
    # on every face, the set of face barycentrics is invariant under the 6 vertex permutations
    lam = np.stack([-(1 + R.r + R.s + R.t) / 2, (1 + R.r) / 2, (1 + R.s) / 2, (1 + R.t) / 2], axis=1)
    for f, verts in enumerate(refelem.FACE_VERTS):
        L = lam[R.Fmask[f]][:, list(verts)]
        for p in itertools.permutations(range(3)):
            Lp = L[:, list(p)]
            a = sorted(map(tuple, np.round(L, 12)))
            b = sorted(map(tuple, np.round(Lp, 12)))
            assert np.allclose(np.array(a), np.array(b), atol=1e-12)


def _random_poly(N, rng):
    """A random polynomial of total degree N in (r, s, t) and its exact gradient."""
    terms = [(a, b, c, rng.normal()) for (a, b, c) in quad.monomials(N)]

    def p(r, s, t):
        return sum(k * r ** a * s ** b * t ** c for a, b, c, k in terms)

    def grad(r, s, t):
        dr = sum(k * a * r ** max(a - 1, 0) * s ** b * t ** c for a, b, c, k in terms if a)
        ds = sum(k * b * r ** a * s ** max(b - 1, 0) * t ** c for a, b, c, k in terms if b)
        dt = sum(k * c * r ** a * s ** b * t ** max(c - 1, 0) for a, b, c, k in terms if c)
        z = 0 * r
        return dr + z, ds + z, dt + z

    return p, grad


def test_derivative_matrices_exact(R):
    rng = np.random.default_rng(R.N)
    assert np.abs(R.Dr @ np.ones(R.Np)).max() < 1e-13
    for _ in range(3):
        p, grad = _random_poly(R.N, rng)
        u = p(R.r, R.s, R.t)
        dr, ds, dt = grad(R.r, R.s, R.t)
        scale = max(1.0, np.abs(u).max())
        assert np.abs(R.Dr @ u - dr).max() < 1e-12 * scale * R.N ** 2
        assert np.abs(R.Ds @ u - ds).max() < 1e-12 * scale * R.N ** 2
        assert np.abs(R.Dt @ u - dt).max() < 1e-12 * scale * R.N ** 2


def test_mass_matrix_by_quadrature(R):
    rng = np.random.default_rng(10 + R.N)
    r, s, t, w = quad.tet_rule(R.N + 3)
    assert abs(np.ones(R.Np) @ R.M @ np.ones(R.Np) - 4.0 / 3.0) < 1e-13
    assert np.allclose(R.M, R.M.T, atol=1e-15)
    assert np.linalg.eigvalsh(R.M).min() > 0
    for _ in range(2):
        p, _ = _random_poly(R.N, rng)
        q, _ = _random_poly(R.N, rng)
        exact = np.sum(w * p(r, s, t) * q(r, s, t))
        disc = p(R.r, R.s, R.t) @ R.M @ q(R.r, R.s, R.t)
        assert abs(disc - exact) < 1e-12 * max(1.0, abs(exact))


def test_lift_reproduces_face_integrals(R):
    """u^T M LIFT_f g = int_{face f} u g  (face parameter measure) for polynomials u, g."""
    rng = np.random.default_rng(20 + R.N)
    u2, v2, w2 = quad.tri_rule(R.N + 3)
    Nfp = R.Nfp
    for f in range(4):
        p, _ = _random_poly(R.N, rng)
        q, _ = _random_poly(R.N, rng)
        fr, fs, ft = quad.face_points(f, u2, v2)
        exact = np.sum(w2 * p(fr, fs, ft) * q(fr, fs, ft))
        g = q(R.r, R.s, R.t)[R.Fmask[f]]
        disc = p(R.r, R.s, R.t) @ R.M @ R.LIFT[:, f * Nfp:(f + 1) * Nfp] @ g
        assert abs(disc - exact) < 1e-11 * max(1.0, abs(exact))
        assert np.allclose(R.Mface[f], R.Mface[f].T, atol=1e-15)
        # face area (parameter measure) = 2
        assert abs(np.ones(Nfp) @ R.Mface[f] @ np.ones(Nfp) - 2.0) < 1e-13


def test_summation_by_parts(R):
    """M Dr + (M Dr)^T = sum_f n_r,f |face f| E_f  (discrete divergence theorem)."""
    Nfp = R.Nfp
    # reference outward normal times (physical area / parameter area) per face
    nr = {0: (0, 0, -1), 1: (0, -1, 0), 2: (1, 1, 1), 3: (-1, 0, 0)}
    for d, D in enumerate((R.Dr, R.Ds, R.Dt)):
        S = R.M @ D
        B = np.zeros((R.Np, R.Np))
        for f in range(4):
            idx = R.Fmask[f]
            B[np.ix_(idx, idx)] += nr[f][d] * R.Mface[f]
        assert np.abs(S + S.T - B).max() < 1e-12 * max(1.0, np.abs(S).max())
