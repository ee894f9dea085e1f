"""Sensor post-processing (§3): oracle pins (what the DFT and
least squares fix: pure tones, constants, Parseval, linearity, power laws, the paper's
percent-of-atmosphere figures) and the product module (paper_1710_03887_b200/analysis.py;
its transform is the library's dg_spectrum kernel) against the oracle's plain DFT sums."""
import math

import numpy as np
import pytest

from oracle import analysis as oan
from paper_1710_03887_b200 import analysis as pan


def test_pure_tone_reads_its_amplitude():
    n, dt, A, k = 256, 0.01, 0.37, 13
    t = np.arange(n) * dt
    p = 1.0 + A * np.cos(2 * np.pi * k * t / (n * dt) + 0.3)
    f, db, a = oan.dft_amplitude(p, dt)
    assert abs(a[k] - A) < 1e-12
    assert np.max(np.delete(a, k)) < 1e-12
    assert abs(f[k] - k / (n * dt)) < 1e-12
    # constant record: every deviation bin is zero -> floored
    f, db, a = oan.dft_amplitude(np.full(64, 1.0), dt)
    assert np.all(db == -200.0)


def test_parseval_and_linearity():
    rng = np.random.default_rng(0)
    n, dt = 200, 0.5
    p = 1.0 + 0.01 * rng.normal(size=n)
    f, db, a = oan.dft_amplitude(p, dt)
    x = p - p.mean()
    # sum x^2 = n/2 * sum a_k^2 over 0<k<n/2, + n a_0^2 + n a_{n/2}^2 (even n)
    e_spec = n * a[0] ** 2 + (n / 2) * (a[1:-1] ** 2).sum() + n * a[-1] ** 2
    assert abs((x * x).sum() - e_spec) < 1e-8 * (x * x).sum()
    f2, db2, a2 = oan.dft_amplitude(1.0 + 3.0 * (p - 1.0), dt)
    nz = a > 1e-14
    assert np.allclose(db2[nz] - db[nz], 20 * math.log10(3.0), atol=1e-9)


def test_decay_exponent_and_percent():
    r = np.array([30.0, 50.0, 80.0, 120.0])
    assert abs(oan.decay_exponent(r, 2.5 / r) + 1.0) < 1e-12
    assert abs(oan.decay_exponent(r, 7.0 / r ** 2) + 2.0) < 1e-12
    # PAPER §3: 400 Pa of 101325 Pa ~ 0.3947 %; 10 Pa ~ 0.009869 %
    assert abs(oan.percent_of_atmosphere(400 / 101325) - 0.3947) < 1e-4   # paper truncates
    assert abs(oan.percent_of_atmosphere(10 / 101325) - 0.009869) < 5e-7
    assert oan.percent_of_atmosphere(0.0) == 0.0


@pytest.mark.gpu
@pytest.mark.parametrize("n", [2, 3, 128, 131, 1000])
def test_product_spectrum_matches_oracle(n):
    rng = np.random.default_rng(n)
    dt, T = 2.9e-3, 1.0 / 340.294
    p = 1.0 + 0.005 * np.exp(-((np.arange(n) - n / 3) / 9.0) ** 2) + 1e-4 * rng.normal(size=n)
    f0, db0, a0 = oan.dft_amplitude(p, dt, T)
    f1, db1, a1 = pan.spectrum(p, dt, T)
    assert np.allclose(f1, f0, rtol=1e-14, atol=0)
    assert np.abs(a1 - a0).max() < 1e-14 * max(1.0, n / 128)
    big = a0 > 1e-10   # dB of round-off-sized bins is not meaningful
    assert np.abs(db1[big] - db0[big]).max(initial=0.0) < 1e-9
    # two sensors at once (columns), and a device-resident record stays on the device
    import torch
    f2, db2, a2 = pan.spectrum(np.stack([p, 2 * p - 1], axis=1), dt, T)
    assert np.abs(a2[:, 1] - 2 * a0).max() < 2e-14 * max(1.0, n / 128)
    xd = torch.as_tensor(np.stack([p, p], axis=1), device="cuda")
    f3, db3, a3 = pan.spectrum(xd, dt, T)
    assert a3.is_cuda and np.abs(a3[:, 0].cpu().numpy() - a1).max() == 0.0
    # a constant record: every bin floored
    f4, db4, a4 = pan.spectrum(np.full(n, 1.25), dt, T)
    assert np.all(a4 < 1e-15)


@pytest.mark.gpu
def test_product_spectrum_pure_tone():
    n, dt, A, k = 256, 0.01, 0.37, 13
    t = np.arange(n) * dt
    p = 1.0 + A * np.cos(2 * np.pi * k * t / (n * dt) + 0.3)
    f, db, a = pan.spectrum(p, dt)
    assert abs(a[k] - A) < 1e-13
    assert np.max(np.delete(a, k)) < 1e-13


def test_product_reflection_decay_percent():
    f = np.linspace(0, 5000, 51)
    near = np.full(51, -40.0)
    d, mean = pan.reflection_indicator(near, near, f, (300, 5000))
    assert mean == 0.0
    d, mean = pan.reflection_indicator(near + 20 * math.log10(2), near, f, (300, 5000))
    assert abs(mean - 6.0206) < 1e-4
    r = np.array([30.0, 50.0, 80.0])
    assert abs(pan.decay_exponent(r, 1 / r) + 1) < 1e-12
    assert abs(pan.percent_of_atmosphere(400 / 101325) - oan.percent_of_atmosphere(400 / 101325)) == 0
    with pytest.raises(ValueError):
        pan.decay_exponent([1, 2], [1, 1])
