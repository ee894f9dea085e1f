"""The oracle's fp64 noise floor (oracle/precision.py):
the extended-precision route is really more precise, and the fp64 floor sits below the
1e-11 RHS parity tolerance (profiles/oracle_noise_floor.json has the full-size values)."""
import mpmath as mp
import numpy as np

from oracle import precision
from oracle.refelem import reference_element
from synth import configs
from synth import mesh as smesh

import parity


def test_extended_geometry_and_operators_are_more_precise():
    m = smesh.kuhn_box((2, 2, 2), (0, 0, 0), (1, 1.1, 0.9))
    v = m.vxyz.copy()
    v += np.random.default_rng(0).uniform(-0.01, 0.01, v.shape)
    g = precision.geometry_longdouble(v, m.etov)
    with mp.workdps(40):
        for k in (0, 7, 31):
            P = [[mp.mpf(float(x)) for x in v[m.etov[k, i]]] for i in range(4)]
            A = mp.matrix([[(P[c + 1][d] - P[0][d]) / 2 for c in range(3)] for d in range(3)])
            J = mp.det(A)
            assert abs(mp.mpf(str(g.J[k])) - J) / J < 1e-18
    R64, RLD = reference_element(3), reference_element(3, np.longdouble)
    d = np.abs(RLD.Dr - R64.Dr.astype(np.longdouble)).max()
    assert 0 < d < 1e-14 and RLD.Dr.dtype == np.longdouble        # rounded differently, same operator


def test_fp64_floor_below_the_parity_tolerance():
    for name, scale in (("C2", 0.25), ("C4", 0.1)):
        cfg = configs.make(name, scale=scale)
        o = parity.oracle_mesh(cfg)
        Q = configs.initial_state(cfg, o.x)
        from oracle.rhs import rhs
        f64 = rhs(o, Q)
        fld = precision.rhs_longdouble(o, Q)
        e = parity.e_rhs(f64, fld.astype(np.float64), parity.scales(cfg))
        assert 1e-17 < e < 1e-12, (name, e)
    # free stream in extended precision: zero to extended round-off
    cfg = configs.make("C5", scale=0.1)
    o = parity.oracle_mesh(cfg)
    Q = np.broadcast_to(np.array([1.3, 0.2, -0.1, 0.3, 3.0])[:, None, None], (5, o.K, o.Np)).copy()
    assert np.abs(precision.rhs_longdouble(o, Q)).max() < 1e-14
