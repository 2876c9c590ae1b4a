"""Quality and timing statistics used by tests and bench (not HyRes arithmetic).

* MPSNR: mean over bands of 10 log10(max(ref_b)^2 / MSE_b) -- SURVEY.md §8(c) Z12
  (the parity metric the north_star's "MPSNR within 0.01 dB" refers to).
* PSNR with a global peak and SAM in radians (PAPER.md:156,
  SPEC.md:292-327) for reporting.
* Olympic mean: drop one fastest and one slowest run (PAPER.md:253-254,
  SPEC.md:510-518).
"""
from __future__ import annotations

import numpy as np


def _as2d(x):
    x = np.asarray(x, dtype=np.float64)
    return x.reshape(x.shape[0], -1)


def mpsnr(ref, est) -> float:
    r, e = _as2d(ref), _as2d(est)
    mse = np.mean((r - e) ** 2, axis=1)
    peak = np.max(r, axis=1) ** 2
    mse = np.maximum(mse, 1e-300)
    return float(np.mean(10.0 * np.log10(peak / mse)))


def psnr(ref, est) -> float:
    r, e = _as2d(ref), _as2d(est)
    mse = max(float(np.mean((r - e) ** 2)), 1e-300)
    return float(10.0 * np.log10(float(np.max(r)) ** 2 / mse))


def sam(ref, est) -> float:
    r, e = _as2d(ref), _as2d(est)
    num = np.sum(r * e, axis=0)
    den = np.linalg.norm(r, axis=0) * np.linalg.norm(e, axis=0)
    ok = den > 0
    cos = np.clip(num[ok] / den[ok], -1.0, 1.0)
    return float(np.mean(np.arccos(cos)))


def rel_l2(ref, est) -> float:
    r = np.asarray(ref, dtype=np.float64).ravel()
    e = np.asarray(est, dtype=np.float64).ravel()
    n = np.linalg.norm(r)
    return float(np.linalg.norm(r - e) / (n if n > 0 else 1.0))


def olympic_mean(values) -> float:
    v = sorted(float(x) for x in values)
    if len(v) < 3:
        raise ValueError("olympic_mean needs at least 3 values")
    return float(np.mean(v[1:-1]))
