"""Pins of the oracle's time integrators.

The LSERK4 coefficients are not in the container; they are
trusted only because the Butcher tableau they imply satisfies the classical
order conditions up to order 4 and its stability polynomial matches exp(z)
through z^4.  Heun (the paper's RK2, P:41 / S:308-316) is checked against its
textbook two-stage form.
"""
import math

import numpy as np
import pytest

from oracle import timestep


def butcher_from_2n(a, b):
    """(A, weights) of the Runge-Kutta method realised by the 2N-storage update."""
    S = len(a)
    A = np.zeros((S + 1, S))        # row s: Y_s = Y_0 + dt sum_j A[s, j] f_j
    Bk = np.zeros(S)                # K_s = dt sum_j Bk[j] f_j
    for s in range(S):
        Bk = a[s] * Bk
        Bk[s] += 1.0
        A[s + 1] = A[s] + b[s] * Bk
    return A[:S], A[S]


def test_lserk4_order_conditions():
    A, w = butcher_from_2n(timestep.LSERK4_A, timestep.LSERK4_B)
    c = A.sum(axis=1)
    assert np.allclose(c, timestep.LSERK4_C, atol=1e-11)       # stage times consistent
    conds = [
        (w.sum(), 1.0),
        (w @ c, 1 / 2),
        (w @ c ** 2, 1 / 3),
        (w @ A @ c, 1 / 6),
        (w @ c ** 3, 1 / 4),
        (w @ (c * (A @ c)), 1 / 8),
        (w @ A @ c ** 2, 1 / 12),
        (w @ A @ A @ c, 1 / 24),
    ]
    for got, want in conds:
        assert got == pytest.approx(want, abs=1e-11)
    # stability polynomial R(z) = 1 + sum_k z^k w^T A^(k-1) 1: matches exp(z) to z^4
    one = np.ones(len(w))
    for k in range(1, 5):
        coef = w @ np.linalg.matrix_power(A, k - 1) @ one
        assert coef == pytest.approx(1 / math.factorial(k), abs=1e-11)


def test_lserk4_linear_amplification():
    lam = -0.7 + 0.4j
    for dt in (0.1, 0.05):
        y, _, _ = timestep.step(lambda q, t: lam * q, np.array([1.0 + 0j]), np.zeros(1, complex), 0.0, dt)
        z = lam * dt
        taylor = sum(z ** k / math.factorial(k) for k in range(5))
        assert abs(y[0] - taylor) < 0.02 * abs(z) ** 5


def test_lserk4_convergence_order_nonlinear():
    # y' = -y^2 + sin t, fixed end time; error ratio under dt halving -> 2^4
    f = lambda y, t: -y * y + np.sin(t)
    def run(n):
        y, _, _ = timestep.integrate(f, np.array([1.0]), 0.0, 1.0 / n, n)
        return y[0]
    ref = run(2048)
    e1, e2 = abs(run(16) - ref), abs(run(32) - ref)
    assert math.log2(e1 / e2) == pytest.approx(4.0, abs=0.3)


def test_heun_is_textbook_heun():
    f = lambda y, t: np.cos(t) * y - y ** 3
    y0, dt, t0 = np.array([0.7]), 0.13, 0.4
    got, _, t1 = timestep.step(f, y0, np.zeros(1), t0, dt, scheme="heun")
    k1 = f(y0, t0)
    k2 = f(y0 + dt * k1, t0 + dt)
    want = y0 + dt / 2 * (k1 + k2)
    assert np.allclose(got, want, atol=1e-16, rtol=0)
    assert t1 == pytest.approx(t0 + dt)
    # one step on y' = z y matches 1 + z + z^2/2
    z = -0.3
    y, _, _ = timestep.step(lambda q, t: z * q, np.array([1.0]), np.zeros(1), 0.0, 1.0, scheme="heun")
    assert y[0] == pytest.approx(1 + z + z * z / 2, abs=1e-16)
