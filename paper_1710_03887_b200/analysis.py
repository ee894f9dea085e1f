"""Post-processing of sensor records: pressure spectra in dB, the
reflection indicator, the amplitude-decay exponent and the percent-of-atmosphere measure
the paper compares domains with (§3; Fig. 5 "the corresponding
pressure pulse in the frequency domain"; "the spectra sampled 1 cm from the boundary
is roughly 1-3 dB larger ... relative to the spectra sampled 2 cm from the boundary";
P:201 "its amplitude will drop off inversely proportional to the distance traveled";
P:257 "a deviation from atmospheric pressure by approximately 0.3947%").

Conventions (reading A22): the ambient (mean) is removed before the transform;
one-sided amplitude spectrum |X_k| = (2/n)|sum_j x_j e^{-2 pi i jk/n}| for 0 < k < n/2
(1/n for k = 0 and the Nyquist bin), so a cosine of amplitude A reads A; dB
relative to 1 scaled pressure unit, floored at -200 dB; frequencies in Hz via the caller's
time scale (seconds per scaled time unit).  The transform runs on the GPU in the library
(`dg_spectrum`, csrc/spectrum.cuh); the rest is small host arithmetic on its output.
"""
from __future__ import annotations

import math

import numpy as np
import torch

from . import dg_spectrum

DB_FLOOR = -200.0


def spectrum(p, dt: float, time_scale: float = 1.0):
    """(freqs_hz, magnitude_db, amplitude) of a uniformly sampled pressure record.

    p: (n,) or (n, m) samples -- a CUDA tensor (e.g. a dg_sensors_record buffer) is transformed
    in place on its device and the results are CUDA tensors; host data (numpy or CPU tensor) is
    copied to the current CUDA device and numpy arrays come back.  dt: sampling interval in
    scaled time units.  freqs are always a host numpy array."""
    on_dev = isinstance(p, torch.Tensor) and p.is_cuda
    x = p if isinstance(p, torch.Tensor) else torch.as_tensor(np.asarray(p, dtype=np.float64))
    if not x.is_cuda:
        if not torch.cuda.is_available():
            raise RuntimeError("spectrum() runs on the GPU (dg_spectrum); no CUDA device available")
        x = x.to("cuda")
    x = x.to(torch.float64).contiguous()
    n = x.shape[0]
    if n < 2:
        raise ValueError("spectrum needs at least two samples")
    m = 1 if x.dim() == 1 else int(np.prod(x.shape[1:]))
    nb = n // 2 + 1
    amp = torch.empty((nb,) + tuple(x.shape[1:]), dtype=torch.float64, device=x.device)
    db = torch.empty_like(amp)
    with torch.cuda.device(x.device):
        st = torch.cuda.current_stream().cuda_stream
        dg_spectrum(x.data_ptr(), n, m, amp.data_ptr(), db.data_ptr(), st)
    freqs = np.arange(nb, dtype=np.float64) / (n * dt * time_scale)
    if on_dev:
        return freqs, db, amp
    torch.cuda.synchronize(x.device)
    return freqs, db.cpu().numpy(), amp.cpu().numpy()


def reflection_indicator(near_db, far_db, freqs, band=(0.0, math.inf)):
    """Per-bin dB difference (near-boundary minus reference sensor) and its mean over `band` (Hz);
    a positive band mean flags a reflection from the boundary.  Host arrays (or tensors)."""
    a = _host(near_db)
    b = _host(far_db)
    f = _host(freqs)
    if a.shape != b.shape or a.shape[0] != f.shape[0]:
        raise ValueError("spectra must share their bin structure")
    d = a - b
    sel = (f >= band[0]) & (f <= band[1])
    return d, float(d[sel].mean()) if bool(sel.any()) else float("nan")


def _host(v):
    if isinstance(v, torch.Tensor):
        v = v.detach().cpu().numpy()
    return np.asarray(v, dtype=np.float64)


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
