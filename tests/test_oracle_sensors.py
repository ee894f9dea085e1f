"""Pins of the oracle's point sensors (oracle/sensors.py, PAPER.md P:220,
Table 2) and the library's host-side sensor location (include/dg.h dg_sensors_set).

The pins fix the sensor arithmetic by what mathematics fixes, independent of either
implementation: the Lagrange weights reproduce the nodal values at the nodes, sum to one
and reproduce every polynomial of degree <= N at arbitrary points; a point built from
known barycentrics in a known element is located there with the same (r,s,t); a linear
pressure field is sampled exactly."""

import numpy as np
import pytest

import paper_1710_03887_b200 as dg
from oracle import geom, sensors
from oracle.refelem import reference_element
from synth import mesh as smesh


@pytest.mark.parametrize("N", [1, 2, 3, 4])
def test_weights_are_lagrange(N):
    R = reference_element(N)
    for i in range(0, R.Np, max(1, R.Np // 6)):
        w = sensors.interp_weights(N, R.r[i], R.s[i], R.t[i])
        e = np.zeros(R.Np)
        e[i] = 1.0
        assert np.abs(w - e).max() < 1e-13
    rng = np.random.default_rng(N)
    # random interior points: partition of unity and exact polynomial reproduction
    exps = [(a, b, c) for a in range(N + 1) for b in range(N + 1 - a) for c in range(N + 1 - a - b)]
    coef = rng.normal(size=len(exps))

    def poly(r, s, t):
        return sum(cf * r ** a * s ** b * t ** c for cf, (a, b, c) in zip(coef, exps))

    for _ in range(5):
        lam = rng.dirichlet(np.ones(4))
        r, s, t = 2 * lam[1] - 1, 2 * lam[2] - 1, 2 * lam[3] - 1
        w = sensors.interp_weights(N, r, s, t)
        assert abs(w.sum() - 1.0) < 1e-13
        assert abs(w @ poly(R.r, R.s, R.t) - poly(r, s, t)) < 1e-12 * max(1.0, np.abs(coef).sum())


def test_locate_known_points():
    m = smesh.kuhn_box((3, 3, 3), (-1, -1, -1), (1, 1, 1))
    V = m.vxyz[m.etov]
    rng = np.random.default_rng(7)
    for k in rng.choice(m.K, 12, replace=False):
        lam = 0.05 + 0.8 * rng.dirichlet(np.ones(4))
        lam /= lam.sum()
        x = lam @ V[k]
        kk, r, s, t = sensors.locate(m.vxyz, m.etov, x)
        assert kk == k
        assert np.allclose([r, s, t], [2 * lam[1] - 1, 2 * lam[2] - 1, 2 * lam[3] - 1], atol=1e-12)
    assert sensors.locate(m.vxyz, m.etov, np.array([1.5, 0.0, 0.0]))[0] == -1
    # a mesh vertex is shared: the smallest containing element wins
    x = m.vxyz[m.etov[40, 0]]
    kk = sensors.locate(m.vxyz, m.etov, x)[0]
    owners = np.nonzero((m.etov == m.etov[40, 0]).any(axis=1))[0]
    assert kk == owners.min()


def test_linear_pressure_field_sampled_exactly():
    """p(x) = 1 + 0.01 x represented exactly -> the sample equals p at the point."""
    N, gamma = 3, 1.4
    m = smesh.kuhn_box((2, 2, 2), (0, 0, 0), (2, 2, 2))
    R = reference_element(N)
    x = geom.node_coordinates(m.vxyz, m.etov, R.r, R.s, R.t)
    p = 1 + 0.01 * x[0]
    Q = np.stack([np.full_like(p, 1.4), 0 * p, 0 * p, 0 * p, p / (gamma - 1)])
    for pt in ([0.3, 1.1, 1.7], [1.9, 0.2, 0.4]):
        k, r, s, t = sensors.locate(m.vxyz, m.etov, np.array(pt))
        out = sensors.sample(N, Q, k, r, s, t, gamma)
        assert abs(out[5] - (1 + 0.01 * pt[0])) < 1e-13
        assert abs(out[0] - 1.4) < 1e-13


def test_library_locates_like_the_oracle():
    """dg_sensors_set's host location (element per point, -1 outside) on an unbound ctx."""
    m = smesh.kuhn_box((3, 2, 2), (-1, -1, -1), (2, 1, 1))
    rng = np.random.default_rng(3)
    pts = np.concatenate([rng.uniform([-1, -1, -1], [2, 1, 1], size=(20, 3)), [[5.0, 0, 0], [-1, -1, -1]]])
    ctx = dg.dg_mesh_create(2, m.vxyz, m.etov, m.bc)
    try:
        el = dg.dg_sensors_set(ctx, pts, 0)
        for p, e in zip(pts, el):
            assert e == sensors.locate(m.vxyz, m.etov, p)[0]
        with pytest.raises(dg.DGError):
            dg.dg_sensors_set(ctx, np.zeros((dg.DG_MAX_SENSORS + 1, 3)), 0)
    finally:
        dg.dg_destroy(ctx)
