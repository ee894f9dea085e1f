"""Post-processing of sensor records: pressure spectra in dB, the
reflection indicator, the amplitude-decay exponent and the percent-of-atmosphere measure
the paper compares domains with (§3; Fig. 5 "the corresponding
pressure pulse in the frequency domain"; "the spectra sampled 1 cm from the boundary
is roughly 1-3 dB larger ... relative to the spectra sampled 2 cm from the boundary";
P:201 "its amplitude will drop off inversely proportional to the distance traveled";
P:257 "a deviation from atmospheric pressure by approximately 0.3947%").

Conventions (reading A22): the ambient (mean) is removed before the transform;
one-sided amplitude spectrum |X_k| = (2/n)|sum_j x_j e^{-2 pi i jk/n}| for 0 < k < n/2
(1/n for k = 0 and the Nyquist bin), so a cosine of amplitude A on bin k reads A; dB
relative to 1 scaled pressure unit, floored at -200 dB; frequencies in Hz via the caller's
time scale (seconds per scaled time unit).  The transforms run where the record lives
(torch.fft, on the GPU for records from dg_sensors_record).
"""
from __future__ import annotations

import math

import numpy as np
import torch

DB_FLOOR = -200.0


def spectrum(p, dt: float, time_scale: float = 1.0):
    """(freqs_hz, magnitude_db, amplitude) of a uniformly sampled pressure record.

    p: (n,) or (n, m) samples (numpy or torch; a torch tensor stays on its device);
    dt: sampling interval in scaled time units."""
    x = p if isinstance(p, torch.Tensor) else torch.as_tensor(np.asarray(p, dtype=np.float64))
    x = x.to(torch.float64)
    n = x.shape[0]
    if n < 2:
        raise ValueError("spectrum needs at least two samples")
    x = x - x.mean(dim=0, keepdim=True)
    X = torch.fft.rfft(x, dim=0)
    amp = X.abs() * (2.0 / n)
    amp[0] = amp[0] / 2
    if n % 2 == 0:
        amp[-1] = amp[-1] / 2
    db = torch.where(amp > 0, 20.0 * torch.log10(amp.clamp_min(1e-300)), torch.full_like(amp, DB_FLOOR))
    db = db.clamp_min(DB_FLOOR)
    freqs = torch.fft.rfftfreq(n, d=dt * time_scale, dtype=torch.float64).to(x.device)
    return freqs, db, amp


def reflection_indicator(near_db, far_db, freqs, band=(0.0, math.inf)):
    """Per-bin dB difference (near-boundary minus reference sensor) and its mean over `band` (Hz);
    a positive band mean flags a reflection from the boundary."""
    a = torch.as_tensor(near_db, dtype=torch.float64)
    b = torch.as_tensor(far_db, dtype=torch.float64, device=a.device)
    f = torch.as_tensor(freqs, dtype=torch.float64, device=a.device)
    if a.shape != b.shape or a.shape[0] != f.shape[0]:
        raise ValueError("spectra must share their bin structure")
    d = a - b
    sel = (f >= band[0]) & (f <= band[1])
    return d, float(d[sel].mean()) if bool(sel.any()) else float("nan")


def decay_exponent(r, dev) -> float:
    """Least-squares slope of log(deviation) against log(distance)."""
    r = np.asarray(r, dtype=np.float64)
    dev = np.asarray(dev, dtype=np.float64)
    if len(r) < 3 or np.any(r <= 0) or np.any(dev <= 0):
        raise ValueError("decay_exponent needs >= 3 positive samples")
    slope, _ = np.polyfit(np.log(r), np.log(dev), 1)
    return float(slope)


def percent_of_atmosphere(deviation, p0: float = 1.0):
    """100 |deviation| / p0 (scaled units: p0 = 1, Eq. 3)."""
    return 100.0 * np.abs(np.asarray(deviation, dtype=np.float64)) / p0
