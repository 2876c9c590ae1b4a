"""HyRes oracle: plain, slow, fp64 CPU implementation of the north_star hot path.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import or call
anything under ``oracle/``.  The product path (``paper_2204_06979_b200``) never
imports it, and the two share no code: this file imports numpy/mpmath only.

What it computes (BASELINE.json north_star stages (1)-(6); SURVEY.md §8(c)
steps C1-C7; every reading of an ambiguous passage is listed in DESIGN.md §2):

C1  G = Y Y^T (uncentered, B x B) over all N = R*C pixels; M = (G + delta I)^-1
    with delta = 1e-6; sigma_b^2 = 1 / (N M_bb) -- the residual variance of the
    least-squares regression of band b on all other bands (HySime's noise
    estimator; "regress band i on all other
    bands ... ridge damping delta=1e-6").
C2  G_w = diag(sigma)^-1 G diag(sigma)^-1 / N; (lambda, V) = eigh(G_w) sorted
    descending; each column of V sign-fixed so its largest-|.| entry is positive,
    lowest index on ties (SPEC.md:181 D6, applied to V).
C3  Daubechies filters by spectral factorisation (SPEC.md:179 D4: Haar, db4,
    db8; default db8 = 16 taps); levels L = max(1, min(5, floor(log2(min(R,C) /
    (taps-1))))).
C4  Eigen-image e_k = (Y^T diag(sigma)^-1 v_k) as an R x C image; L-level
    separable periodised orthonormal 2-D DWT, each level first padding an odd
    extent by duplicating the last row/column (SPEC.md:182 D7); along an axis of
    even length n: a_j = sum_m h_m x_{(2j+m) mod n}, d_j = sum_m g_m x_{(2j+m) mod n}
    (SPEC.md:118-126).
C5  Per subband (noise sigma = 1 in whitened units): SURE threshold
    t* = a_(k*), k* = smallest argmin_k S_k, S_k = n - 2k + sum_{i<=k} a_(i)^2
    + (n-k) a_(k)^2 over the sorted |x| with a_(0) = 0 (north_star stage (5):
    "sort, prefix sums, argmin"); then soft threshold sign(x) max(|x|-t*, 0)
    (SPEC.md:136-137).
C6  Rank: E_post,k = sum of soft(x)^2 over all subbands of component k, N_c its
    coefficient count; walking k = 1, 2, ...: the first k with E_post,k <= N_c
    stops the walk and r* = max(1, k-1); r* = B if none fails (SPEC.md:380 step
    (5) "retain components whose post-threshold energy exceeds a noise-floor
    criterion").
C7  e^_k = IDWT(soft coefficients) (the adjoint synthesis, cropping each level's
    padding); X^ = sum_{k<=r*} (sigma (.) v_k) e^_k^T, returned as float32 BSQ
    (SPEC.md:380 step (6) "inverse transforms and de-whitening").

F1  (NEXT row of SURVEY.md §8(f)) HySime subspace identification: R_y = Y Y^T/N,
    R_n = N~ N~^T/N from the band-by-band regression residual N~, R_x = R_y - R_n
    = E diag(mu) E^T, delta_i = -e_i^T R_y e_i + 2 e_i^T R_n e_i, k = #{delta_i < 0}
    (SPEC.md:370-377), pinned by tests/test_oracle_pins.py::test_f1_*.

Parity pins for every function are in tests/test_oracle_*.py (SURVEY.md §8(c)
P1-P8).  P9 (the paper's Houston anchor) is "parity unpinned":
the data is not available.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

DEFAULT_RIDGE = 1e-6          # SPEC.md:364 "ridge damping delta=1e-6"
DEFAULT_TAPS = 16             # SPEC.md:179 D4 "default Daubechies-8"
SUPPORTED_TAPS = (2, 8, 16)   # Haar, db4, db8 (SPEC.md:179 D4)
MAX_AUTO_LEVELS = 5
HYSIME_TOL = 1e-9             # DESIGN.md R13: |delta_i| below this x max p_j counts as zero


# ----------------------------------------------------------------------------
# C3: filters
# ----------------------------------------------------------------------------
def daubechies_lowpass(n_moments: int, dps: int = 50) -> np.ndarray:
    """Daubechies minimum-phase scaling filter with `n_moments` vanishing moments
    (2*n_moments taps), by spectral factorisation (Daubechies, Ten Lectures §6.1):
    |H(w)|^2 = 2 cos^{2N}(w/2) P(sin^2(w/2)), P(y) = sum_{k<N} C(N-1+k, k) y^k.
    Each root y_i of P gives z + 1/z = 2 - 4 y_i; the root z_i with |z_i| < 1 is
    kept (minimum phase), H(z) ~ (1 + z)^N prod_i (z - z_i).  Normalised so
    sum h = sqrt(2); ordered so h_0 is the coefficient of the highest power
    (energy front-loaded; h_0 = 0.0544158... for N = 8)."""
    import mpmath as mp
    N = int(n_moments)
    if N < 1:
        raise ValueError("n_moments >= 1")
    if N == 1:
        return np.array([1.0, 1.0]) / math.sqrt(2.0)
    with mp.workdps(dps):
        # polyroots wants highest-degree coefficient first
        coeffs = [mp.binomial(N - 1 + k, k) for k in range(N - 1, -1, -1)]
        yroots = mp.polyroots(coeffs, maxsteps=200, extraprec=4 * dps)
        zs = []
        for y in yroots:
            c = 1 - 2 * y                      # z^2 - 2c z + 1 = 0
            s = mp.sqrt(c * c - 1)
            z1, z2 = c + s, c - s
            zs.append(z1 if abs(z1) < 1 else z2)
        poly = [mp.mpc(1)]                     # coefficients, highest power first
        for _ in range(N):
            poly = _polymul(poly, [mp.mpc(1), mp.mpc(1)])
        for z in zs:
            poly = _polymul(poly, [mp.mpc(1), -z])
        re = [mp.re(p) for p in poly]
        tot = mp.fsum(re)
        h = [p * mp.sqrt(2) / tot for p in re]
        return np.array([float(v) for v in h])


def _polymul(a, b):
    out = [0] * (len(a) + len(b) - 1)
    for i, x in enumerate(a):
        for j, y in enumerate(b):
            out[i + j] += x * y
    return out


def filters(taps: int = DEFAULT_TAPS):
    """(h, g): analysis low/high-pass, g_k = (-1)^k h_{T-1-k} (quadrature mirror)."""
    if taps not in SUPPORTED_TAPS:
        raise ValueError(f"taps must be one of {SUPPORTED_TAPS}")
    h = daubechies_lowpass(taps // 2)
    T = len(h)
    g = np.array([(-1.0) ** k * h[T - 1 - k] for k in range(T)])
    return h, g


def auto_levels(rows: int, cols: int, taps: int = DEFAULT_TAPS) -> int:
    """L = max(1, min(5, floor(log2(min(R, C) / (taps - 1))))) -- DESIGN.md reading R6."""
    m = min(rows, cols)
    v = m / max(taps - 1, 1)
    lv = int(math.floor(math.log2(v))) if v >= 1 else 0
    return max(1, min(MAX_AUTO_LEVELS, lv))


def level_shapes(rows: int, cols: int, levels: int):
    """Subband shape per level 1..L: (ceil(h/2), ceil(w/2)) of the previous level's LL."""
    shapes = []
    h, w = rows, cols
    for _ in range(levels):
        h, w = (h + 1) // 2, (w + 1) // 2
        shapes.append((h, w))
    return shapes


def check_levels(rows: int, cols: int, levels: int):
    if levels < 1 or min(rows, cols) < 2 ** levels:
        raise ValueError("levels impossible for this image size (SPEC.md:122)")


def coeff_count(rows: int, cols: int, levels: int) -> int:
    """N_c: coefficients of one eigen-image = 3 sum_l h_l w_l + h_L w_L."""
    sh = level_shapes(rows, cols, levels)
    return 3 * sum(h * w for h, w in sh) + sh[-1][0] * sh[-1][1]


# ----------------------------------------------------------------------------
# C4: DWT (periodised, per-level symmetric pad-to-even)
# ----------------------------------------------------------------------------
def _pad_even(x: np.ndarray, axis: int) -> np.ndarray:
    if x.shape[axis] % 2 == 0:
        return x
    last = np.take(x, [x.shape[axis] - 1], axis=axis)
    return np.concatenate([x, last], axis=axis)


def analysis_1d(x: np.ndarray, h: np.ndarray, g: np.ndarray, axis: int):
    """a_j = sum_m h_m x_{(2j+m) mod n}, d_j = sum_m g_m x_{(2j+m) mod n}; n even."""
    x = np.moveaxis(np.asarray(x, dtype=np.float64), axis, -1)
    n = x.shape[-1]
    assert n % 2 == 0
    j2 = 2 * np.arange(n // 2)
    a = np.zeros(x.shape[:-1] + (n // 2,))
    d = np.zeros_like(a)
    for m in range(len(h)):
        xm = x[..., (j2 + m) % n]
        a += h[m] * xm
        d += g[m] * xm
    return np.moveaxis(a, -1, axis), np.moveaxis(d, -1, axis)


def synthesis_1d(a: np.ndarray, d: np.ndarray, h: np.ndarray, g: np.ndarray, axis: int):
    """Adjoint of analysis_1d: x_i = sum_{j,m: (2j+m) mod n = i} h_m a_j + g_m d_j."""
    a = np.moveaxis(np.asarray(a, dtype=np.float64), axis, -1)
    d = np.moveaxis(np.asarray(d, dtype=np.float64), axis, -1)
    half = a.shape[-1]
    n = 2 * half
    x = np.zeros(a.shape[:-1] + (n,))
    j2 = 2 * np.arange(half)
    for m in range(len(h)):
        idx = (j2 + m) % n
        contrib = h[m] * a + g[m] * d
        if len(np.unique(idx)) == len(idx):
            x[..., idx] += contrib
        else:  # filter longer than the signal: several taps wrap onto one sample
            for jj in range(half):
                x[..., idx[jj]] += contrib[..., jj]
    return np.moveaxis(x, -1, axis)


SUBBANDS = ("LH", "HL", "HH")   # (axis-0 filter, axis-1 filter): L=lowpass, H=highpass


def dwt2(img: np.ndarray, levels: int, taps: int = DEFAULT_TAPS):
    """Returns {'details': [(LH, HL, HH) for level 1..L], 'LL': LL_L, 'shapes': [...]}.
    Level l: pad the current LL to even, filter along axis 1 (columns, contiguous),
    then along axis 0."""
    h, g = filters(taps)
    x = np.asarray(img, dtype=np.float64)
    check_levels(x.shape[0], x.shape[1], levels)
    details, in_shapes = [], []
    for _ in range(levels):
        in_shapes.append(x.shape)
        x = _pad_even(_pad_even(x, 0), 1)
        lo1, hi1 = analysis_1d(x, h, g, axis=1)
        ll, hl = analysis_1d(lo1, h, g, axis=0)      # axis0 L / H of the axis1-lowpass
        lh, hh = analysis_1d(hi1, h, g, axis=0)      # axis0 L / H of the axis1-highpass
        details.append((lh, hl, hh))
        x = ll
    return {"details": details, "LL": x, "in_shapes": in_shapes}


def idwt2(coeffs, taps: int = DEFAULT_TAPS) -> np.ndarray:
    """Inverse of dwt2: per level from coarsest, synthesise along axis 0 then axis 1,
    then crop that level's padding."""
    h, g = filters(taps)
    x = coeffs["LL"]
    for (lh, hl, hh), shp in zip(reversed(coeffs["details"]), reversed(coeffs["in_shapes"])):
        lo1 = synthesis_1d(x, hl, h, g, axis=0)
        hi1 = synthesis_1d(lh, hh, h, g, axis=0)
        x = synthesis_1d(lo1, hi1, h, g, axis=1)
        x = x[: shp[0], : shp[1]]
    return x


def flatten_coeffs(coeffs) -> List[np.ndarray]:
    """Subbands in the storage order used at the C-ABI: level 1..L x (LH, HL, HH), then LL_L."""
    out = []
    for lh, hl, hh in coeffs["details"]:
        out += [lh, hl, hh]
    out.append(coeffs["LL"])
    return out


def unflatten_coeffs(subbands: List[np.ndarray], template):
    lv = len(template["details"])
    det = [tuple(subbands[3 * i: 3 * i + 3]) for i in range(lv)]
    return {"details": det, "LL": subbands[-1], "in_shapes": template["in_shapes"]}


# ----------------------------------------------------------------------------
# C5: SURE
# ----------------------------------------------------------------------------
@dataclass
class SureResult:
    k: int              # index into {0} U sorted |x| (k = 0 means t = 0)
    t: float            # threshold a_(k)
    risk: float         # S_k
    margin: float       # second-best S minus best S (tie diagnostics)


def sure_threshold(x: np.ndarray) -> SureResult:
    """k* = smallest argmin over k = 0..n of S_k = n - 2k + sum_{i<=k} a_(i)^2 + (n-k) a_(k)^2,
    a = sorted |x|, a_(0) = 0 (noise sigma = 1)."""
    a = np.sort(np.abs(np.asarray(x, dtype=np.float64).ravel()))
    n = a.size
    a0 = np.concatenate([[0.0], a])
    k = np.arange(n + 1, dtype=np.float64)
    csum = np.concatenate([[0.0], np.cumsum(a * a)])
    s = n - 2.0 * k + csum + (n - k) * a0 * a0
    kstar = int(np.argmin(s))
    best = s[kstar]
    rest = np.delete(s, kstar)
    margin = float(np.min(rest) - best) if rest.size else float("inf")
    return SureResult(kstar, float(a0[kstar]), float(best), margin)


def sure_risk_direct(x: np.ndarray, t: float) -> float:
    """S(t) = n - 2 #{|x_i| <= t} + sum_i min(x_i^2, t^2) (Stein's unbiased risk, sigma = 1)."""
    ax = np.abs(np.asarray(x, dtype=np.float64).ravel())
    return float(ax.size - 2.0 * np.count_nonzero(ax <= t) + np.sum(np.minimum(ax * ax, t * t)))


def soft_threshold(x: np.ndarray, t: float) -> np.ndarray:
    """sign(x) max(|x| - t, 0)."""
    if t < 0:
        raise ValueError("t >= 0")
    x = np.asarray(x, dtype=np.float64)
    return np.sign(x) * np.maximum(np.abs(x) - t, 0.0)


# ----------------------------------------------------------------------------
# C1: noise estimate
# ----------------------------------------------------------------------------
def _as_bands_by_pixels(cube: np.ndarray) -> np.ndarray:
    cube = np.asarray(cube)
    if cube.ndim != 3:
        raise ValueError("cube must be (bands, rows, cols) BSQ")
    if not np.all(np.isfinite(cube)):
        raise FloatingPointError("non-finite input (SPEC.md:26)")
    return cube.reshape(cube.shape[0], -1).astype(np.float64)


def gram(cube: np.ndarray) -> np.ndarray:
    """G = Y Y^T over all pixels (uncentered), fp64."""
    y = _as_bands_by_pixels(cube)
    return y @ y.T


def estimate_noise(cube: np.ndarray, ridge: float = DEFAULT_RIDGE, want_residual: bool = False):
    """sigma (B,), G (B,B) [, residual (B,R,C)] with sigma_b^2 = 1/(N M_bb), M = (G + ridge I)^-1.
    residual_b = (M Y)_b / M_bb -- the regression residual of band b on the others."""
    b, r, c = np.asarray(cube).shape
    n = r * c
    if b < 3 or n <= b:
        raise ValueError("bands >= 3 and pixels > bands required (SPEC.md:363, :365)")
    y = _as_bands_by_pixels(cube)
    g = y @ y.T
    m = np.linalg.inv(g + ridge * np.eye(b))
    sigma = np.sqrt(1.0 / (n * np.diag(m)))
    if want_residual:
        res = (m @ y) / np.diag(m)[:, None]
        return sigma, g, res.reshape(b, r, c)
    return sigma, g


# ----------------------------------------------------------------------------
# C2: whitening + eigendecomposition
# ----------------------------------------------------------------------------
def sign_fix(v: np.ndarray) -> np.ndarray:
    """Flip each column so its largest-|.| entry (lowest index on ties) is positive."""
    v = v.copy()
    for j in range(v.shape[1]):
        i = int(np.argmax(np.abs(v[:, j])))
        if v[i, j] < 0:
            v[:, j] = -v[:, j]
    return v


def whiten_eig(g: np.ndarray, sigma: np.ndarray, n: int):
    gw = g / np.outer(sigma, sigma) / n
    lam, v = np.linalg.eigh(gw)
    order = np.argsort(-lam, kind="stable")
    return lam[order], sign_fix(v[:, order]), gw


# ----------------------------------------------------------------------------
# full path
# ----------------------------------------------------------------------------
@dataclass
class HyresResult:
    out: np.ndarray                 # float32 BSQ
    rank: int
    levels: int
    sigma: np.ndarray
    gram: np.ndarray
    lam: np.ndarray
    V: np.ndarray
    n_coeffs: int
    e_post: List[float] = field(default_factory=list)
    sure: List[List[SureResult]] = field(default_factory=list)   # per visited component, per subband
    eigen_images: List[np.ndarray] = field(default_factory=list) # e_k before the DWT (visited ones)
    denoised_images: List[np.ndarray] = field(default_factory=list)  # e^_k for k <= r*


def hyres(cube: np.ndarray, taps: int = DEFAULT_TAPS, levels: int = 0, ridge: float = DEFAULT_RIDGE,
          keep_ll: bool = False, keep_images: bool = False) -> HyresResult:
    cube = np.asarray(cube)
    b, r, c = cube.shape
    n = r * c
    lv = levels if levels > 0 else auto_levels(r, c, taps)
    check_levels(r, c, lv)
    sigma, g = estimate_noise(cube, ridge)                                    # C1
    lam, v, _ = whiten_eig(g, sigma, n)                                       # C2
    y = _as_bands_by_pixels(cube)
    nc = coeff_count(r, c, lv)
    e_post, sure_all, eimgs, kept = [], [], [], []
    for k in range(b):                                                        # C6 walk
        w = v[:, k] / sigma
        ek = (w @ y).reshape(r, c)                                            # C4 projection
        co = dwt2(ek, lv, taps)
        subs = flatten_coeffs(co)
        res_k, soft = [], []
        for si, sb in enumerate(subs):                                        # C5
            if keep_ll and si == len(subs) - 1:
                sr = SureResult(0, 0.0, float("nan"), float("inf"))
            else:
                sr = sure_threshold(sb)
            res_k.append(sr)
            soft.append(soft_threshold(sb, sr.t))
        ep = float(sum(np.sum(s * s) for s in soft))
        e_post.append(ep)
        sure_all.append(res_k)
        if keep_images:
            eimgs.append(ek)
        if ep <= nc and k > 0:
            break
        kept.append(idwt2(unflatten_coeffs(soft, co), taps))                  # C7 IDWT
        if ep <= nc:       # k == 0 failed: r* = max(1, 0) keeps component 1
            break
    rank = len(kept)
    u = v[:, :rank] * sigma[:, None]                                          # D^{1/2} V
    ehat = np.stack([e.ravel() for e in kept])                                # (r*, N)
    out = (u @ ehat).reshape(b, r, c).astype(np.float32)                      # C7
    return HyresResult(out, rank, lv, sigma, g, lam, v, nc, e_post, sure_all,
                       eimgs, kept if keep_images else [])


# ----------------------------------------------------------------------------
# F1: HySime subspace identification
# ----------------------------------------------------------------------------
@dataclass
class HysimeResult:
    k: int                  # signal subspace dimension: #{i : delta_i < 0}
    basis: np.ndarray       # B x k, eigenvectors of R_x in ascending-delta order (D6 signs)
    delta: np.ndarray       # (B,) delta_i = -p_i + 2 sigma_i^2, in the order of mu (descending)
    mu: np.ndarray          # (B,) eigenvalues of R_x, descending
    E: np.ndarray           # B x B eigenvectors of R_x (columns, descending mu, D6 signs)
    noise_cov: np.ndarray   # R_n = N~^T N~ / N (B x B)
    r_y: np.ndarray         # R_y = Y Y^T / N


def noise_residual(cube: np.ndarray, ridge: float = DEFAULT_RIDGE) -> np.ndarray:
    """N~ (B x N): residual of the least-squares regression of every band on all
    the other bands, N~_b = y_b - Y_{-b} beta_b, written out
    band by band from the normal equations with the ridge of S:364 on the
    other-band block.  Slow (B solves); small cubes only."""
    y = _as_bands_by_pixels(cube)
    b = y.shape[0]
    g = y @ y.T
    res = np.empty_like(y)
    for i in range(b):
        o = [j for j in range(b) if j != i]
        a = g[np.ix_(o, o)] + ridge * np.eye(b - 1)
        beta = np.linalg.solve(a, g[o, i])
        res[i] = y[i] - beta @ y[o]
    return res


def hysime(cube: np.ndarray, ridge: float = DEFAULT_RIDGE) -> HysimeResult:
    """HySime ("eigendecompose the signal correlation estimate
    (R_y - R_n), select dimension k minimizing the sum of projection-error and
    noise-power terms"; the criterion of Bioucas-Dias & Nascimento, HySime, which
    HyDe implements):
      R_y = Y Y^T / N;  R_n = N~ N~^T / N with N~ the regression residual
      (noise_residual, SPEC.md:364 post: noise_cov = (1/N) N~^T N~);
      R_x = R_y - R_n = E diag(mu) E^T (mu descending, D6 signs);
      p_i = e_i^T R_y e_i, sigma_i^2 = e_i^T R_n e_i, delta_i = -p_i + 2 sigma_i^2
      (the mean-square-error change of adding e_i to the subspace: minus the
      projected signal power plus twice the projected noise power);
      the error sum over a subspace is minimised by taking exactly the
      eigenvectors with delta_i < 0: k = #{delta_i < 0}, basis = those
      eigenvectors in ascending-delta order (stable on ties).
    Reading (R13): a delta_i within 1e-9 max_j p_j of zero counts as
    non-negative -- on a noiseless cube the null-space eigenvectors carry
    p_i ~ sigma_i^2 ~ rounding and their sign is noise (SPEC.md:375 expects
    k == 1 for a noiseless rank-1 cube)."""
    y = _as_bands_by_pixels(cube)
    b, n = y.shape
    if b < 3 or n <= b:
        raise ValueError("bands >= 3 and pixels > bands required (SPEC.md:363, :365)")
    r_y = (y @ y.T) / n
    res = noise_residual(cube, ridge)
    r_n = (res @ res.T) / n
    r_x = r_y - r_n
    mu, e = np.linalg.eigh(0.5 * (r_x + r_x.T))
    order = np.argsort(-mu, kind="stable")
    mu, e = mu[order], sign_fix(e[:, order])
    p = np.einsum("ij,ik,kj->j", e, r_y, e)
    s2 = np.einsum("ij,ik,kj->j", e, r_n, e)
    delta = -p + 2.0 * s2
    asc = np.argsort(delta, kind="stable")
    tol = HYSIME_TOL * float(np.max(np.abs(p)))
    k = int(np.count_nonzero(delta < -tol))
    return HysimeResult(k, e[:, asc[:k]], delta, mu, e, r_n, r_y)


# ----------------------------------------------------------------------------
# F2: FORPDN
# ----------------------------------------------------------------------------
FORPDN_GRID = (0.1, 1.0, 10.0, 100.0)   # SPEC.md:432 D16


def spectral_difference(b: int) -> np.ndarray:
    """D ((b-1) x b): first-order spectral difference, (D x)_i = x_{i+1} - x_i."""
    d = np.zeros((b - 1, b))
    for i in range(b - 1):
        d[i, i] = -1.0
        d[i, i + 1] = 1.0
    return d


@dataclass
class ForpdnResult:
    out: np.ndarray         # float32 BSQ
    lam: float
    residual_power: dict    # lambda -> ||W - X(lambda)||_F^2 / (N B)
    noise_power: float      # trace(R_n) / B (HySime's noise estimate)


def forpdn(cube: np.ndarray, lam: Optional[float] = None, taps: int = DEFAULT_TAPS, levels: int = 0,
           ridge: float = DEFAULT_RIDGE) -> ForpdnResult:
    """FORPDN (SPEC.md:388-396 D16; "full-rank, wavelet-based"):
    W (N_c x B) = per-band 2-D DWT coefficients (the C4 transform of every band
    image); X = argmin ||W - X||_F^2 + lam ||X D^T||_F^2 = W (I + lam D^T D)^-1
    (one B x B solve for every coefficient row); the output is the per-band
    inverse DWT of X.  Default lam (SPEC.md:432 D16): from {0.1, 1, 10, 100},
    the one whose residual power ||W - X||^2 / (N B) is closest to HySime's
    noise power trace(R_n) / B (first on ties) -- reading R14: the residual is
    taken in the coefficient domain (equal to the image-domain residual by
    Parseval when 2^L divides R and C)."""
    cube = np.asarray(cube)
    b, r, c = cube.shape
    if b < 2:
        raise ValueError("bands >= 2 required (SPEC.md:392)")
    lv = levels or auto_levels(r, c, taps)
    check_levels(r, c, lv)
    tmpl = dwt2(np.zeros((r, c)), lv, taps)
    rows = [np.concatenate([s.ravel() for s in flatten_coeffs(dwt2(cube[i].astype(np.float64), lv, taps))])
            for i in range(b)]
    w = np.stack(rows, axis=1)                          # N_c x B
    d = spectral_difference(b)
    n = r * c

    def solve(lmb):
        a = np.eye(b) + lmb * (d.T @ d)
        return w @ np.linalg.inv(a)                     # X = W A^-1 (A symmetric)

    res_pow, noise_pow = {}, None
    if lam is None:
        res = noise_residual(cube, ridge)
        noise_pow = float(np.trace(res @ res.T) / n / b)
        best = None
        for lmb in FORPDN_GRID:
            x = solve(lmb)
            rp = float(np.sum((w - x) ** 2) / (n * b))
            res_pow[lmb] = rp
            if best is None or abs(rp - noise_pow) < abs(res_pow[best] - noise_pow):
                best = lmb
        lam = best
    if not lam > 0:
        raise ValueError("lambda > 0 required (SPEC.md:392)")
    x = solve(lam)
    sizes = [s.size for s in flatten_coeffs(tmpl)]
    offs = np.cumsum([0] + sizes)
    out = np.empty((b, r, c))
    for i in range(b):
        subs = [x[offs[j]:offs[j + 1], i].reshape(flatten_coeffs(tmpl)[j].shape) for j in range(len(sizes))]
        out[i] = idwt2(unflatten_coeffs(subs, tmpl), taps)
    return ForpdnResult(out.astype(np.float32), float(lam), res_pow, noise_pow)


# ----------------------------------------------------------------------------
# F4: WSRRR
# ----------------------------------------------------------------------------
@dataclass
class WsrrrResult:
    out: np.ndarray             # float32 BSQ denoised cube
    components: np.ndarray      # float32 (rank, R, C): inverse DWT of the columns of C
    V: np.ndarray               # B x rank, column-orthonormal
    objective: List[float]      # per sweep
    lam: float
    rank: int


def band_dwt_matrix(cube: np.ndarray, levels: int, taps: int) -> np.ndarray:
    """W (N_c x B): the C4 DWT of every band image, one column per band."""
    cols = [np.concatenate([s.ravel() for s in flatten_coeffs(dwt2(cube[i].astype(np.float64), levels, taps))])
            for i in range(cube.shape[0])]
    return np.stack(cols, axis=1)


def band_idwt_matrix(x: np.ndarray, rows: int, cols: int, levels: int, taps: int) -> np.ndarray:
    """Inverse of band_dwt_matrix for the columns of x (N_c x m) -> (m, R, C)."""
    tmpl = dwt2(np.zeros((rows, cols)), levels, taps)
    shapes = [s.shape for s in flatten_coeffs(tmpl)]
    offs = np.cumsum([0] + [int(np.prod(sh)) for sh in shapes])
    out = np.empty((x.shape[1], rows, cols))
    for i in range(x.shape[1]):
        subs = [x[offs[j]:offs[j + 1], i].reshape(shapes[j]) for j in range(len(shapes))]
        out[i] = idwt2(unflatten_coeffs(subs, tmpl), taps)
    return out


def wsrrr(cube: np.ndarray, rank: Optional[int] = None, lam: Optional[float] = None, max_iters: int = 20,
          tol: float = 1e-4, taps: int = DEFAULT_TAPS, levels: int = 0, ridge: float = DEFAULT_RIDGE) -> WsrrrResult:
    """WSRRR (SPEC.md:397-405 D17; §2.1 "Wavelet-Based Sparse Reduced-Rank
    Regression"): min_{C,V} ||W - C V^T||_F^2 + lam ||C||_1 s.t. V^T V = I, with W
    (N_c x B) the per-band DWT coefficients.  Alternating: C = soft(W V, lam/2)
    (the exact minimiser over C for orthonormal V, since ||W - C V^T||^2 =
    ||W V - C||^2 + const); V = P Q^T from the SVD P S Q^T = W^T C (orthogonal
    Procrustes).  Readings (R15): V_0 = the top-rank eigenvectors of
    W^T W (D6 signs); one sweep = C-step then V-step, the objective evaluated
    after the sweep; stop when |f_prev - f| <= tol f_prev or after max_iters
    sweeps; default rank = HySime's k (at least 1); default lam (D17) =
    sigma^ sqrt(2 ln N_c), sigma^ = sqrt(mean_b sigma_b^2) from estimate_noise.
    Output: inverse DWT of C V^T per band; components: inverse DWT of the
    columns of C."""
    cube = np.asarray(cube)
    b, r, c = cube.shape
    lv = levels or auto_levels(r, c, taps)
    check_levels(r, c, lv)
    if rank is None:
        rank = max(1, hysime(cube, ridge).k)
    if rank < 1 or rank > b:
        raise ValueError("1 <= rank <= bands required (SPEC.md:401)")
    w = band_dwt_matrix(cube, lv, taps)
    nc = w.shape[0]
    if lam is None:
        sigma, _ = estimate_noise(cube, ridge)
        lam = float(np.sqrt(np.mean(sigma ** 2)) * np.sqrt(2.0 * np.log(nc)))
    if lam < 0:
        raise ValueError("lambda >= 0 required")
    g = w.T @ w
    mu, e = np.linalg.eigh(g)
    order = np.argsort(-mu, kind="stable")
    v = sign_fix(e[:, order])[:, :rank]
    obj = []
    cmat = None
    for _ in range(max_iters):
        cmat = soft_threshold(w @ v, lam / 2.0)
        m = w.T @ cmat
        p, _, qt = np.linalg.svd(m, full_matrices=False)
        v = p @ qt
        f = float(np.sum((w - cmat @ v.T) ** 2) + lam * np.sum(np.abs(cmat)))
        obj.append(f)
        if len(obj) > 1 and abs(obj[-2] - obj[-1]) <= tol * obj[-2]:
            break
    out = band_idwt_matrix(cmat @ v.T, r, c, lv, taps)
    comps = band_idwt_matrix(cmat, r, c, lv, taps)
    return WsrrrResult(out.astype(np.float32), comps.astype(np.float32), v, obj, float(lam), int(rank))


# ----------------------------------------------------------------------------
# F3: HyMiNoR
# ----------------------------------------------------------------------------
def shrink(v: np.ndarray, t: float) -> np.ndarray:
    """sign(v) max(|v| - t, 0)."""
    return np.sign(v) * np.maximum(np.abs(v) - t, 0.0)


@dataclass
class L1SpecResult:
    out: np.ndarray             # float32 BSQ
    iters: np.ndarray           # (N,) iterations run per pixel
    residuals: List[float]      # Bregman residual ||x - m - a||^2 + ||D x - d||^2 (all pixels) per iteration


def l1_spectral(m_cube: np.ndarray, lam: float = 10.0, mu: float = 5.0, max_iters: int = 50,
                tol: float = 1e-3) -> L1SpecResult:
    """Second stage of HyMiNoR (SPEC.md:415-423 D19; §2.1 "the remaining
    sparse noise is removed by solving an l1-l1 optimization problem with a
    modified split-Bregman technique"): per pixel spectrum m (length B),
    min_x ||m - x||_1 + lam ||D x||_1, D the first-order spectral difference, by
    split Bregman with a = x - m, d = D x:
      x = (I + D^T D)^-1 (a + m - b_a + D^T (d - b_d))
      a = shrink(x - m + b_a, 1/mu),  b_a += x - m - a
      d = shrink(D x + b_d, lam/mu),   b_d += D x - d
    from x = m, a = d = b_a = b_d = 0 (reading R16); a pixel stops when
    ||x_new - x_old|| <= tol ||x_old|| or after max_iters."""
    b, r, c = m_cube.shape
    m = np.asarray(m_cube, dtype=np.float64).reshape(b, -1)
    n = m.shape[1]
    dmat = spectral_difference(b)
    ainv = np.linalg.inv(np.eye(b) + dmat.T @ dmat)
    x = m.copy()
    a = np.zeros_like(m)
    ba = np.zeros_like(m)
    d = np.zeros((b - 1, n))
    bd = np.zeros((b - 1, n))
    active = np.ones(n, dtype=bool)
    iters = np.zeros(n, dtype=np.int64)
    resid = []
    for _ in range(max_iters):
        if not active.any():
            break
        idx = np.nonzero(active)[0]
        xo = x[:, idx]
        rhs = a[:, idx] + m[:, idx] - ba[:, idx] + dmat.T @ (d[:, idx] - bd[:, idx])
        xn = ainv @ rhs
        t = xn - m[:, idx] + ba[:, idx]
        an = shrink(t, 1.0 / mu)
        ba[:, idx] = t - an
        a[:, idx] = an
        u = dmat @ xn + bd[:, idx]
        dn = shrink(u, lam / mu)
        bd[:, idx] = u - dn
        d[:, idx] = dn
        x[:, idx] = xn
        iters[idx] += 1
        resid.append(float(np.sum((x - m - a) ** 2) + np.sum((dmat @ x - d) ** 2)))
        done = np.sqrt(np.sum((xn - xo) ** 2, axis=0)) <= tol * np.sqrt(np.sum(xo ** 2, axis=0))
        active[idx[done]] = False
    return L1SpecResult(x.reshape(b, r, c).astype(np.float32), iters, resid)


def hyminor(cube: np.ndarray, lam: float = 10.0, mu: float = 5.0, max_iters: int = 50, tol: float = 1e-3):
    """HyMiNoR (SPEC.md:415-423 D19): M = hyres(cube), then l1_spectral(M)."""
    if not (lam > 0 and mu > 0):
        raise ValueError("lambda, mu > 0 required (SPEC.md:420)")
    return l1_spectral(hyres(cube).out, lam, mu, max_iters, tol)
