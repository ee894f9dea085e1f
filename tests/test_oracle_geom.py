"""Pins of the oracle's geometry and connectivity."""
import math

import numpy as np
import pytest

from oracle import conn, geom
from synth import mesh as smesh

UNIT = np.array([[0.0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]])


def test_unit_tet_examples():
    g = geom.geometric_factors(UNIT, np.array([[0, 1, 2, 3]]))
    assert g.volume[0] == pytest.approx(1 / 6, abs=1e-15)
    # face f2 = (v2 v3 v4) is opposite the origin: n = (1,1,1)/sqrt3, area sqrt3/2
    assert np.allclose(g.nx[0, 2], np.ones(3) / math.sqrt(3), atol=1e-15)
    assert g.area[0, 2] == pytest.approx(math.sqrt(3) / 2, abs=1e-15)
    assert np.allclose(g.nx[0, 0], [0, 0, -1]) and g.area[0, 0] == pytest.approx(0.5)
    assert np.allclose(g.nx[0, 1], [0, -1, 0]) and np.allclose(g.nx[0, 3], [-1, 0, 0])
    g2 = geom.geometric_factors(2 * UNIT, np.array([[0, 1, 2, 3]]))
    assert g2.volume[0] == pytest.approx(8 / 6)
    assert np.allclose(g2.area, 4 * g.area)
    assert g.h[0] == pytest.approx(3 * (1 / 6) / (math.sqrt(3) / 2))


def test_degenerate_rejected():
    flat = np.array([[0.0, 0, 0], [1, 0, 0], [0, 1, 0], [1, 1, 0]])
    with pytest.raises(ValueError):
        geom.geometric_factors(flat, np.array([[0, 1, 2, 3]]))


def test_invariants_on_random_mesh():
    m = smesh.kuhn_box((3, 3, 3), (0, 0, 0), (1, 1, 1))
    rng = np.random.default_rng(0)
    v = m.vxyz + rng.uniform(-0.05, 0.05, m.vxyz.shape)
    g = geom.geometric_factors(v, m.etov)
    assert np.abs(np.linalg.norm(g.nx, axis=2) - 1).max() < 1e-12
    closed = (g.area[:, :, None] * g.nx).sum(axis=1)
    assert np.abs(closed).max() < 1e-10
    etoe, etof = conn.connect_by_hashing(m.etov)
    inter = ~conn.is_boundary(etoe, etof)
    k, f = np.nonzero(inter)
    assert np.allclose(g.nx[k, f], -g.nx[etoe[k, f], etof[k, f]], atol=1e-12)


def test_adjacency_counts():
    e, f = conn.connect_by_hashing(np.array([[0, 1, 2, 3]]))
    assert conn.is_boundary(e, f).sum() == 4
    e, f = conn.connect_by_hashing(np.array([[0, 1, 2, 3], [1, 2, 3, 4]]))
    b = conn.is_boundary(e, f)
    assert b.sum() == 6 and (~b).sum() == 2                                # 1 interior face
    m = smesh.kuhn_box((4, 3, 2), (0, 0, 0), (1, 1, 1))
    e, f = conn.connect_by_hashing(m.etov)
    b = conn.is_boundary(e, f).sum()
    assert ((~conn.is_boundary(e, f)).sum()) // 2 == (4 * m.K - b) // 2
    assert b == 2 * 2 * (4 * 3 + 3 * 2 + 4 * 2)                            # 2 tris per boundary quad
    conn.check_symmetric(e, f)
    with pytest.raises(ValueError):
        conn.connect_by_hashing(np.array([[0, 1, 2, 3], [0, 1, 2, 4], [0, 1, 2, 5]]))


def test_vmaps_pair_coincident_nodes_including_periodic():
    from oracle.refelem import reference_element
    R = reference_element(3)
    m = smesh.kuhn_box((3, 3, 3), (0, 0, 0), (1, 1, 1), periodic=(True, True, True))
    g = geom.geometric_factors(m.vxyz, m.etov)
    x = geom.node_coordinates(m.vxyz, m.etov, R.r, R.s, R.t)
    vM, vP = conn.build_vmaps(x, m.vxyz, m.etov, m.etoe, m.etof, R.Fmask, g.h)
    X = x.reshape(3, -1)
    d = X[:, vM] - X[:, vP]
    d = d - np.round(d)                         # unit-period minimum image
    assert np.abs(d).max() < 1e-12
    # the pairing is an involution: the neighbour's trace of my trace is me
    Np = R.Np
    for k in range(0, m.K, 7):
        for f in range(4):
            k2, f2 = m.etoe[k, f], m.etof[k, f]
            for i in range(R.Nfp):
                i2 = int(np.nonzero(vM[k2, f2] == vP[k, f, i])[0][0])
                assert vP[k2, f2, i2] == vM[k, f, i]
    assert vM.max() < m.K * Np
