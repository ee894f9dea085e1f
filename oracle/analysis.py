"""Oracle sensor post-processing: amplitude spectrum, reflection
indicator, decay exponent, percent of atmosphere.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Definitions written out (reading A22; §3, Fig. 5):
  x_j = p_j - mean(p);  X_k = sum_j x_j (cos(2 pi jk/n) - i sin(2 pi jk/n))  (plain DFT sum)
  amplitude a_k = 2|X_k|/n for 0 < k < n/2, |X_k|/n for k = 0 and k = n/2;  f_k = k/(n dt T)
  dB = 20 log10(a_k / 1), floored at -200;  reflection = dB_near - dB_ref, mean over a band;
  decay exponent = least-squares slope of log(dev) on log(r) (normal equations);
  percent of atmosphere = 100 |dev| / p0.
"""
from __future__ import annotations

import numpy as np


def dft_amplitude(p, dt: float, time_scale: float = 1.0):
    x = np.asarray(p, dtype=np.float64)
    n = len(x)
    x = x - x.sum() / n
    k = np.arange(n // 2 + 1)
    j = np.arange(n)
    ang = 2.0 * np.pi * np.outer(k, j) / n
    re = (np.cos(ang) * x).sum(axis=1)
    im = -(np.sin(ang) * x).sum(axis=1)
    a = 2.0 * np.sqrt(re * re + im * im) / n
    a[0] /= 2
    if n % 2 == 0:
        a[-1] /= 2
    f = k / (n * dt * time_scale)
    with np.errstate(divide="ignore"):
        db = np.where(a > 0, 20.0 * np.log10(a), -200.0)
    return f, np.maximum(db, -200.0), a


def decay_exponent(r, dev) -> float:
    X = np.log(np.asarray(r, dtype=np.float64))
    Y = np.log(np.asarray(dev, dtype=np.float64))
    n = len(X)
    sx, sy, sxx, sxy = X.sum(), Y.sum(), (X * X).sum(), (X * Y).sum()
    return float((n * sxy - sx * sy) / (n * sxx - sx * sx))


def percent_of_atmosphere(dev, p0: float = 1.0):
    return 100.0 * np.abs(np.asarray(dev, dtype=np.float64)) / p0
