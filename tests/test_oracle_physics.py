"""Pins of the oracle's pointwise physics.

Values are SPEC's worked examples and the
paper's printed constants (Eq. 3; pulse amplitude P:181; sensor
amplitudes P:257), each cited at its assertion.
"""
import math

import numpy as np
import pytest

from oracle import euler

G = 1.4
REST = np.array([1.4, 0.0, 0.0, 0.0, 2.5])       # Eq. 3


def test_pressure_examples():
    # S:269-271
    assert euler.pressure(np.array([1.4, 0, 0, 0, 2.5]), G) == pytest.approx(1.0, abs=1e-15)
    assert euler.pressure(np.array([1.4, 1.4, 0, 0, 3.2]), G) == pytest.approx(1.0, abs=1e-15)
    assert euler.pressure(np.array([2.8, 0, 0, 0, 5.0]), G) == pytest.approx(2.0, abs=1e-15)


def test_flux_examples():
    # rest state -> F_x = (0,1,0,0,0), F_y = (0,0,1,0,0); this pins reading A1
    F, Gy, H = euler.euler_fluxes(REST, G)
    assert np.allclose(F, [0, 1, 0, 0, 0], atol=1e-15)
    assert np.allclose(Gy, [0, 0, 1, 0, 0], atol=1e-15)
    assert np.allclose(H, [0, 0, 0, 1, 0], atol=1e-15)
    # u = 1, rho = 1.4, p = 1 -> F_x = (1.4, 2.4, 0, 0, 4.2)
    q = np.array([1.4, 1.4, 0, 0, 1.0 / 0.4 + 0.5 * 1.4])
    F, _, _ = euler.euler_fluxes(q, G)
    assert np.allclose(F, [1.4, 2.4, 0, 0, 4.2], atol=1e-14)


def test_flux_rotation_covariance():
    # n.F(q) must rotate with the momentum -- the garbled "rho v w + p" of Eq. 1 would not
    rng = np.random.default_rng(0)
    Rm, _ = np.linalg.qr(rng.normal(size=(3, 3)))
    q = np.array([1.3, 0.2, -0.3, 0.45, 2.9])
    n = np.array([0.3, -0.5, 0.8]) / np.linalg.norm([0.3, -0.5, 0.8])
    qr = q.copy()
    qr[1:4] = Rm @ q[1:4]
    f = euler.normal_flux(q, n, G)
    fr = euler.normal_flux(qr, Rm @ n, G)
    assert np.allclose(fr[[0, 4]], f[[0, 4]], atol=1e-14)
    assert np.allclose(fr[1:4], Rm @ f[1:4], atol=1e-14)


def test_llf_examples_and_properties():
    n = np.array([0.6, 0.0, 0.8])
    # equal ambient states -> (0, nx, ny, nz, 0), lambda = c = 1
    assert np.allclose(euler.llf_flux(REST, REST, n, G), [0, 0.6, 0, 0.8, 0], atol=1e-15)
    assert euler.llf_lambda(REST, REST, n, G) == pytest.approx(1.0, abs=1e-15)
    assert euler.sound_speed(REST, G) == pytest.approx(1.0, abs=1e-15)       # c0 = 1
    rng = np.random.default_rng(1)
    for _ in range(10):
        a = np.array([1.4, 0, 0, 0, 2.5]) + rng.uniform(-0.1, 0.1, 5)
        b = np.array([1.4, 0, 0, 0, 2.5]) + rng.uniform(-0.1, 0.1, 5)
        m = rng.normal(size=3)
        m /= np.linalg.norm(m)
        # consistency
        assert np.allclose(euler.llf_flux(a, a, m, G), euler.normal_flux(a, m, G), atol=1e-14)
        # conservation / antisymmetry
        assert np.allclose(euler.llf_flux(a, b, m, G), -euler.llf_flux(b, a, -m, G), atol=1e-14)


def test_wall_ghost_examples():
    # S:396-398
    q = np.array([1.4, 1.4 * 0.3, 1.4 * 0.1, 0.0, 3.0])
    g = euler.ghost_wall(q, np.array([1.0, 0, 0]))
    assert np.allclose(g[1:4] / g[0], [-0.3, 0.1, 0.0], atol=1e-15)
    q = np.array([1.4, 1.4, 0.0, 0.0, 3.2])
    nn = np.array([1.0, 1.0, 0]) / math.sqrt(2)
    g = euler.ghost_wall(q, nn)
    assert np.allclose(g[1:4] / g[0], [0.0, -1.0, 0.0], atol=1e-15)   # mirror reading A2
    # the printed component-wise form of Eq. 4 would give (-0.414, 0, 0) here
    assert not np.allclose(g[1:4] / g[0], [1 - 2 / math.sqrt(2), 0, 0], atol=1e-3)
    # involution, |v|, rho, p, E preserved
    rng = np.random.default_rng(2)
    for _ in range(5):
        q = np.array([1.2, 0.3, -0.2, 0.5, 3.1])
        m = rng.normal(size=3)
        m /= np.linalg.norm(m)
        g = euler.ghost_wall(q, m)
        assert np.allclose(euler.ghost_wall(g, m), q, atol=1e-15)
        assert g[0] == q[0] and g[4] == q[4]
        assert np.linalg.norm(g[1:4]) == pytest.approx(np.linalg.norm(q[1:4]), rel=1e-15)
        assert euler.pressure(g, G) == pytest.approx(euler.pressure(q, G), rel=1e-14)
        # no mass or energy crosses a wall
        fs = euler.llf_flux(q, g, m, G)
        assert abs(fs[0]) < 1e-14 and abs(fs[4]) < 1e-14


def test_passthrough_ghost():
    # returns the Eq. 3 state whatever the interior
    q = np.array([[1.0, 2.0], [0.1, 0.2], [0.0, 0.3], [0.0, 0.0], [3.0, 4.0]])
    g = euler.ghost_passthrough(q, REST)
    assert np.allclose(g, REST[:, None])


def test_inflow_ghost_and_pulse():
    # S:415 (recomputed in SURVEY §4): at the peak p = 1.1
    g = euler.ghost_inflow(1.1, G)
    rho = g[0]
    assert rho == pytest.approx(1.4986294, abs=5e-8)
    assert g[1] / rho == pytest.approx(0.0714286, abs=5e-8)
    assert g[4] == pytest.approx(2.753823, abs=5e-7)
    # the pulse p1 peaks at 1.1 at t = pi/alpha and is 1 after 2 pi/alpha
    alpha = 565.0
    assert float(euler.inflow_pressure(math.pi / alpha, alpha)) == pytest.approx(1.1, abs=1e-15)
    assert float(euler.inflow_pressure(2 * math.pi / alpha + 1e-9, alpha)) == 1.0
    assert float(euler.inflow_pressure(0.0, alpha)) == pytest.approx(1.0, abs=1e-15)


def test_inflow_state_generalises_the_printed_eq7():
    """Reading A24: at the paper's constants (Eq. 3 ambient, a = 0.05, time in the units alpha
    is given in) the q_inf-relative inflow state is exactly the printed Eq. 7 (P:206-216:
    rho = gamma p^(1/gamma), u = (p - p0)/(rho0 c)) applied to p1 of P:173-181."""
    alpha = 565.0
    for t in (0.0, 0.3 / alpha, math.pi / alpha, 5.9 / alpha, 2 * math.pi / alpha + 1e-9):
        want = euler.ghost_inflow(euler.inflow_pressure(t, alpha), G)
        got = euler.inflow_state(t, REST, G, alpha=alpha, time_scale=1.0)
        assert np.allclose(got, want, rtol=1e-14, atol=1e-15)
    # another ambient state: the ghost is the same pulse in those units (p0 scales, c0 follows)
    q2 = np.array([1.225, 0.0, 0.0, 0.0, 101325.0 / 0.4])
    g2 = euler.inflow_state(math.pi / alpha, q2, G, alpha=alpha, time_scale=1.0)
    p2 = euler.pressure(g2, G)
    assert p2 == pytest.approx(1.1 * 101325.0, rel=1e-14)                 # peak p0 (1 + 2a)
    c0 = math.sqrt(G * 101325.0 / 1.225)
    assert g2[1] / g2[0] == pytest.approx(0.1 * 101325.0 / (1.225 * c0), rel=1e-14)   # Eq. 5
    assert g2[0] == pytest.approx(1.225 * 1.1 ** (1 / G), rel=1e-14)                  # Eq. 6


def test_inflow_pulse_duration_in_scaled_time():
    """alpha = 565 rad per physical second, time_scale = 1 cm / 343 m/s
    = 2.915e-5 s per scaled unit, so the pulse lasts 2 pi / 565 s = 11.12 ms = 381.5 scaled units."""
    tau = 2.915e-5
    dur = 2 * math.pi / (565.0 * tau)
    assert 0.01 / 343.0 == pytest.approx(tau, rel=2e-4)
    assert 2 * math.pi / 565.0 == pytest.approx(11.12e-3, rel=1e-3)
    assert dur == pytest.approx(381.5, abs=0.1)
    peak = euler.inflow_state(dur / 2, REST, G)                # default alpha, tau, a
    assert euler.pressure(peak, G) == pytest.approx(1.1, rel=1e-12)
    after = euler.inflow_state(dur * 1.0001, REST, G)
    assert np.allclose(after, REST, rtol=0, atol=1e-15)


def test_paper_constants():
    # Eq. 3: p0 = 1, rho0 = 1.4 give c0 = 1 and E0 = 2.5
    assert euler.pressure(REST, G) == pytest.approx(1.0)
    assert math.sqrt(G * 1.0 / 1.4) == pytest.approx(1.0)
    # 10 % pulse = 10132.5 Pa ("approximately 10,000 Pa"); P:257 percentages
    assert 0.1 * 101325 == pytest.approx(10132.5)
    assert 400 / 101325 * 100 == pytest.approx(0.3947, abs=1e-4)   # paper truncates
    assert 10 / 101325 * 100 == pytest.approx(0.009869, abs=5e-7)
