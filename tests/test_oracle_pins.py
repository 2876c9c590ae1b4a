"""Pins for the fp64 oracle: each checks oracle/hyres_ref.py
against something other than itself -- brute force, closed forms, textbook identities,
an independent LAPACK routine, SPEC.md worked examples or invariances that follow from
the method's definition -- chosen so that a dropped term, wrong sign/index or
transposed operand fails at least one of them."""
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest

from oracle import hyres_ref as O
from harness import synth, metrics


# ---------------------------------------------------------------- P1 noise estimator
def _regress_residuals(y):
    """Explicit least squares of each band on all the others (brute force, lstsq)."""
    b, n = y.shape
    res = np.empty_like(y)
    for i in range(b):
        others = np.delete(y, i, axis=0).T          # (N, B-1)
        beta, *_ = np.linalg.lstsq(others, y[i], rcond=None)
        res[i] = y[i] - others @ beta
    return res


def test_p1_noise_equals_explicit_regression_no_ridge():
    rng = np.random.default_rng(1)
    b, r, c = 8, 20, 25
    mix = rng.standard_normal((b, b))
    cube = (mix @ rng.standard_normal((b, r * c))).reshape(b, r, c)
    sig, g, res = O.estimate_noise(cube, ridge=0.0, want_residual=True)
    brute = _regress_residuals(cube.reshape(b, -1))
    sig_brute = np.sqrt(np.sum(brute ** 2, axis=1) / (r * c))
    assert np.max(np.abs(sig / sig_brute - 1)) < 1e-10
    assert np.max(np.abs(res.reshape(b, -1) - brute)) / np.max(np.abs(brute)) < 1e-10
    assert np.allclose(g, cube.reshape(b, -1) @ cube.reshape(b, -1).T, rtol=1e-14)


def test_p1_default_ridge_is_negligible_on_scaled_data():
    rng = np.random.default_rng(2)
    b, n = 12, 600
    y = 10.0 * (rng.standard_normal((b, b)) @ rng.standard_normal((b, n)))
    sig, _ = O.estimate_noise(y.reshape(b, 20, 30))
    brute = _regress_residuals(y)
    sig_brute = np.sqrt(np.sum(brute ** 2, axis=1) / n)
    assert np.max(np.abs(sig / sig_brute - 1)) < 1e-8


def test_p1_parameter_errors(golden_dir):
    ex = json.load(open(os.path.join(golden_dir, "spec_examples.json")))["noise_too_few_bands"]
    with pytest.raises(ValueError):
        O.estimate_noise(np.ones((ex["bands"], ex["rows"], ex["cols"])))
    with pytest.raises(ValueError):            # pixels <= bands
        O.estimate_noise(np.random.default_rng(0).standard_normal((10, 3, 3)))
    with pytest.raises(FloatingPointError):    # non-finite
        bad = np.ones((4, 8, 8)); bad[1, 2, 3] = np.nan
        O.estimate_noise(bad)


# ---------------------------------------------------------------- P2 pure-noise sigma
def test_p2_pure_gaussian_noise_sigma_recovered():
    """RSS_b ~ sigma_b^2 chi^2_{N-B+1}  =>  E[sigma_hat^2] = sigma^2 (N-B+1)/N; every band within 2 %."""
    rng = np.random.default_rng(3)
    b, r, c = 32, 256, 256
    n = r * c
    s = rng.uniform(0.5, 2.0, size=b)
    cube = (s[:, None] * rng.standard_normal((b, n))).reshape(b, r, c)
    sig, _ = O.estimate_noise(cube)
    ratio = sig ** 2 / (s ** 2 * (n - b + 1) / n)
    assert np.max(np.abs(ratio - 1)) < 0.02
    assert abs(np.mean(ratio) - 1) < 0.005


def test_p2_spec_examples_noise():
    """rank-3 noiseless cube -> tiny noise; white noise sigma^2 within 20 % (64x64x30)."""
    rng = np.random.default_rng(4)
    b, r, c = 30, 64, 64
    lr = rng.uniform(0, 1, (b, 3)) @ rng.uniform(0, 1, (3, r * c))
    sig, _ = O.estimate_noise(lr.reshape(b, r, c))
    assert np.sum(sig ** 2) <= 1e-3 * np.mean(lr ** 2)
    s0 = 0.05
    sig2, _ = O.estimate_noise((lr + s0 * rng.standard_normal(lr.shape)).reshape(b, r, c))
    # regression on noisy regressors over-estimates by ~sigma^2 ||beta||^2 (errors in variables),
    # so the SPEC's 20 % holds for the band mean; single bands are allowed 25 %
    ratio = sig2 ** 2 / s0 ** 2
    assert abs(np.mean(ratio) - 1) < 0.2 and np.all(np.abs(ratio - 1) < 0.25) and np.all(ratio > 0.95)


# ---------------------------------------------------------------- P4 filters
def test_p4_db2_closed_form(golden_dir):
    gd = json.load(open(os.path.join(golden_dir, "db2_closed_form.json")))
    want = np.array([eval(e, {"sqrt": math.sqrt}) for e in gd["h_expr"]])
    got = O.daubechies_lowpass(gd["n_moments"])
    assert np.max(np.abs(got - want)) < 1e-15
    h8, _ = O.filters(16)
    assert abs(h8[0] - gd["db8_h0_leading_digits"]["value"]) < gd["db8_h0_leading_digits"]["abs_tol"]


@pytest.mark.parametrize("taps", [2, 8, 16])
def test_p4_filter_identities(taps):
    h, g = O.filters(taps)
    T, N = len(h), taps // 2
    assert T == taps
    assert abs(np.sum(h) - math.sqrt(2)) < 1e-14
    for m in range(T // 2):                      # double-shift orthonormality
        assert abs(np.dot(h[: T - 2 * m], h[2 * m:]) - (1.0 if m == 0 else 0.0)) < 1e-14
        assert abs(np.dot(g[: T - 2 * m], g[2 * m:]) - (1.0 if m == 0 else 0.0)) < 1e-14
    for m in range(-(T // 2) + 1, T // 2):       # h _|_ shifted g
        acc = sum(h[k] * g[k + 2 * m] for k in range(T) if 0 <= k + 2 * m < T)
        assert abs(acc) < 1e-14
    k = np.arange(T, dtype=np.float64)
    for p in range(N):                           # N vanishing moments of the high-pass
        scale = np.sum(np.abs(k ** p * g))
        assert abs(np.sum(k ** p * g)) < 1e-13 * scale
    # minimum phase: after dividing sum_n h_n z^{T-1-n} by (1+z)^N (exactly divisible:
    # N zeros at z=-1) the remaining zeros lie inside the unit circle
    if T > 2:
        q, rem = np.polydiv(h, np.poly(-np.ones(N)))
        assert np.max(np.abs(rem)) < 1e-12
        assert np.all(np.abs(np.roots(q)) < 1.0)


def test_p4_unknown_wavelet():
    with pytest.raises(ValueError):
        O.filters(6)


# ---------------------------------------------------------------- P3 DWT
SHAPES = [(64, 64), (145, 145), (61, 34), (35, 95), (32, 48), (17, 33)]


@pytest.mark.parametrize("taps", [2, 8, 16])
@pytest.mark.parametrize("shape", SHAPES)
def test_p3_perfect_reconstruction_and_parseval(taps, shape):
    rng = np.random.default_rng(5)
    x = rng.standard_normal(shape)
    L = max(1, min(3, int(math.log2(min(shape))) - 1))
    co = O.dwt2(x, L, taps)
    y = O.idwt2(co, taps)
    assert y.shape == x.shape
    assert np.max(np.abs(y - x)) < 1e-12 * max(1.0, np.max(np.abs(x)))
    # per-level Parseval on the padded input of that level
    cur = x
    for lev in range(L):
        one = O.dwt2(cur, 1, taps)
        padded = O._pad_even(O._pad_even(cur, 0), 1)
        e_in = np.sum(padded ** 2)
        e_out = np.sum(one["LL"] ** 2) + sum(np.sum(s ** 2) for s in one["details"][0])
        assert abs(e_out - e_in) < 1e-12 * e_in
        # the multi-level transform's level-(lev+1) details are this single-level transform's
        for a, b in zip(co["details"][lev], one["details"][0]):
            assert np.max(np.abs(a - b)) < 1e-12 * max(1.0, np.max(np.abs(b)))
        cur = one["LL"]


def test_p3_periodised_transform_is_orthogonal_matrix():
    """Build the analysis matrix column by column on an even 16x12 image: W W^T = I."""
    r, c = 16, 12
    cols = []
    for i in range(r * c):
        e = np.zeros(r * c); e[i] = 1.0
        co = O.dwt2(e.reshape(r, c), 2, 16)
        cols.append(np.concatenate([s.ravel() for s in O.flatten_coeffs(co)]))
    w = np.array(cols).T
    assert w.shape == (r * c, r * c)
    assert np.max(np.abs(w @ w.T - np.eye(r * c))) < 1e-13


def test_p3_haar_constant_and_level_errors(golden_dir):
    gd = json.load(open(os.path.join(golden_dir, "spec_examples.json")))
    ex = gd["haar_constant"]
    co = O.dwt2(np.full((ex["rows"], ex["cols"]), ex["c"]), ex["levels"], ex["taps"])
    assert np.allclose(co["LL"], ex["approx"], atol=1e-15)
    for s in co["details"][0]:
        assert np.allclose(s, ex["detail"], atol=1e-15)
    # same for db8: constants live in the approximation only (vanishing moments), LL = 2c
    co8 = O.dwt2(np.full((32, 32), ex["c"]), 1, 16)
    assert np.allclose(co8["LL"], 2 * ex["c"], atol=1e-13)
    for s in co8["details"][0]:
        assert np.allclose(s, 0.0, atol=1e-13)
    t = gd["too_many_levels"]
    with pytest.raises(ValueError):
        O.dwt2(np.zeros((t["rows"], t["cols"])), t["levels"], 2)


def test_p3_unit_coefficient_atom_and_linearity():
    rng = np.random.default_rng(6)
    x = rng.standard_normal((32, 32))
    co = O.dwt2(x, 2, 16)
    subs = O.flatten_coeffs(co)
    for si in range(len(subs)):
        z = [np.zeros_like(s) for s in subs]
        z[si].flat[3] = 1.0
        atom = O.idwt2(O.unflatten_coeffs(z, co), 16)
        assert abs(np.sum(atom ** 2) - 1.0) < 1e-12
    zero = O.idwt2(O.unflatten_coeffs([np.zeros_like(s) for s in subs], co), 16)
    assert np.all(zero == 0)
    y = rng.standard_normal((32, 32))
    a, b = 0.7, -1.3
    lhs = O.flatten_coeffs(O.dwt2(a * x + b * y, 2, 16))
    r1 = O.flatten_coeffs(O.dwt2(x, 2, 16)); r2 = O.flatten_coeffs(O.dwt2(y, 2, 16))
    for l, p, q in zip(lhs, r1, r2):
        assert np.max(np.abs(l - (a * p + b * q))) < 1e-12


def test_p3_auto_levels_and_counts():
    want = {"tiny": 2, "small": 3, "medium": 4, "wide": 4, "large": 5, "batched": 4}
    for name, lv in want.items():
        cfg = synth.CONFIGS[name]
        assert O.auto_levels(cfg.rows, cfg.cols, 16) == lv
    assert O.coeff_count(145, 145, 3) == 21538          # SURVEY.md §8(a) A4 example
    assert O.coeff_count(1024, 1024, 5) == 1024 * 1024


# ---------------------------------------------------------------- P5 SURE
def _brute_sure(x):
    """Exact (rational) S(t) for every candidate t in {0} U {|x_i|}; returns (best_t, best_S)."""
    xs = [Fraction(v) for v in np.abs(x).tolist()]
    n = len(xs)
    best = None
    for t in sorted(set([Fraction(0)] + xs)):
        s = n - 2 * sum(1 for v in xs if v <= t) + sum(min(v * v, t * t) for v in xs)
        if best is None or s < best[1]:
            best = (t, s)
    return best


def test_p5_sure_equals_brute_force_exact():
    rng = np.random.default_rng(7)
    for trial in range(300):
        n = int(rng.integers(1, 65))
        kind = trial % 3
        if kind == 0:
            x = rng.standard_normal(n) * rng.uniform(0.3, 4)
        elif kind == 1:   # duplicates and zeros on a dyadic grid (exact arithmetic)
            x = rng.integers(-8, 9, size=n) / 4.0
        else:             # sparse spikes + noise
            x = rng.standard_normal(n); x[rng.random(n) < 0.2] *= 10
        res = O.sure_threshold(x)
        bt, bs = _brute_sure(x)
        assert res.t == float(bt), (trial, res, bt)
        assert abs(res.risk - float(bs)) <= 1e-9 * (n + float(np.sum(x * x)))
        assert abs(O.sure_risk_direct(x, res.t) - res.risk) <= 1e-9 * (n + float(np.sum(x * x)))
        # no threshold on a dense grid beats the argmin
        grid = np.linspace(0, np.max(np.abs(x)) * 1.2 + 1e-9, 400)
        assert min(O.sure_risk_direct(x, t) for t in grid) >= res.risk - 1e-9 * (n + float(np.sum(x * x)))


def test_p5_sure_special_cases():
    assert O.sure_threshold(np.zeros(10)).t == 0.0                 # all zero -> t = 0, S = -n
    assert O.sure_threshold(np.zeros(10)).risk == -10.0
    big = np.array([100.0, -200.0, 300.0])                       # all large -> keep everything
    assert O.sure_threshold(big).t == 0.0
    small = np.full(1000, 0.01)                                  # all tiny -> kill everything
    r = O.sure_threshold(small)
    assert r.t == pytest.approx(0.01) and O.soft_threshold(small, r.t).max() == 0.0


def test_soft_threshold_spec_examples(golden_dir):
    gd = json.load(open(os.path.join(golden_dir, "spec_examples.json")))["soft_threshold"]
    for x, t, want in gd["cases"]:
        assert O.soft_threshold(np.array([x]), t)[0] == want
    with pytest.raises(ValueError):
        O.soft_threshold(np.array([1.0]), -1.0)


# ---------------------------------------------------------------- P4' eigensolver
def test_p4_whiten_eig_against_independent_svd():
    s = synth.make_cube("tiny", 0)
    b, r, c = s.noisy.shape
    n = r * c
    sig, g = O.estimate_noise(s.noisy)
    lam, v, gw = O.whiten_eig(g, sig, n)
    assert np.all(np.diff(lam) <= 0)
    assert np.max(np.abs(v.T @ v - np.eye(b))) < 1e-12
    assert np.max(np.abs(gw @ v - v * lam)) < 1e-12 * lam[0]
    for j in range(b):
        i = int(np.argmax(np.abs(v[:, j])))
        assert v[i, j] > 0
    # singular values of the whitened data matrix (gesdd, a different LAPACK path)
    yw = s.noisy.reshape(b, -1).astype(np.float64) / sig[:, None] / math.sqrt(n)
    sv = np.linalg.svd(yw, compute_uv=False)
    assert np.max(np.abs(sv ** 2 - lam) / lam[0]) < 1e-12


# ---------------------------------------------------------------- P6 invariances
@pytest.fixture(scope="module")
def tiny_case():
    s = synth.make_cube("tiny", 0)
    return s, O.hyres(s.noisy)


def test_p6_band_permutation(tiny_case):
    s, ref = tiny_case
    perm = np.random.default_rng(8).permutation(s.noisy.shape[0])
    out = O.hyres(s.noisy[perm]).out
    assert metrics.rel_l2(ref.out[perm], out) < 1e-6   # float32 output rounding


def test_p6_transpose(tiny_case):
    s, ref = tiny_case
    out = O.hyres(np.ascontiguousarray(s.noisy.transpose(0, 2, 1))).out
    assert metrics.rel_l2(ref.out.transpose(0, 2, 1), out) < 1e-6


def test_p6_circular_shift_by_multiple_of_2L(tiny_case):
    s, ref = tiny_case
    assert ref.levels == 2
    sh = np.roll(s.noisy, (12, -8), axis=(1, 2))
    out = O.hyres(sh).out
    assert metrics.rel_l2(np.roll(ref.out, (12, -8), axis=(1, 2)), out) < 1e-6
    # negative control: a 1-pixel shift is NOT an invariance of the decimated DWT
    out1 = O.hyres(np.roll(s.noisy, 1, axis=2)).out
    assert metrics.rel_l2(np.roll(ref.out, 1, axis=2), out1) > 1e-4


def test_p6_band_scaling(tiny_case):
    s, ref = tiny_case
    cs = np.random.default_rng(9).uniform(0.5, 2.0, s.noisy.shape[0]).astype(np.float32)
    scaled = (s.noisy * cs[:, None, None]).astype(np.float32)
    out = O.hyres(scaled).out
    assert metrics.rel_l2(ref.out * cs[:, None, None], out) < 1e-6


def test_p6_exact_invariance_fp64_path(tiny_case):
    """Same invariance without the float32 output rounding: reconstruct in fp64 by hand."""
    s, ref = tiny_case
    perm = np.random.default_rng(10).permutation(s.noisy.shape[0])
    r2 = O.hyres(s.noisy[perm], keep_images=True)
    r1 = O.hyres(s.noisy, keep_images=True)
    x1 = (r1.V[:, :r1.rank] * r1.sigma[:, None]) @ np.stack([e.ravel() for e in r1.denoised_images])
    x2 = (r2.V[:, :r2.rank] * r2.sigma[:, None]) @ np.stack([e.ravel() for e in r2.denoised_images])
    assert metrics.rel_l2(x1[perm], x2) < 1e-12


# ---------------------------------------------------------------- P7 / P8
def test_p7_noiseless_low_rank_recovered():
    """Noiseless rank-r cube: r* = r and X^ = X up to the ridge floor.  sigma_b^2 -> delta/N when
    G is singular, so SURE works at noise level sqrt(delta/N) ~ 1.6e-5 here and the residual
    error scales with delta (reading R3): ~3e-6 at delta = 1e-6, ~3e-8 at 1e-9."""
    for seed in (11, 12):
        s = synth.low_rank_cube(64, 64, 32, rank=4, seed=seed)
        res = O.hyres(s.clean)
        assert res.rank == 4
        assert metrics.rel_l2(s.clean, res.out) < 1e-5
        assert metrics.psnr(s.clean, res.out) >= 45.0
        fine = O.hyres(s.clean, ridge=1e-9)
        assert fine.rank == 4
        assert metrics.rel_l2(s.clean, fine.out) < 1e-7


def test_p8_denoising_gain_tiny(tiny_case):
    s, ref = tiny_case
    gain = metrics.mpsnr(s.clean, ref.out) - metrics.mpsnr(s.clean, s.noisy)
    assert gain >= 10.0
    assert metrics.sam(s.clean, ref.out) < metrics.sam(s.clean, s.noisy)


def test_p8_spec_rank6_example():
    """synthetic rank-6 cube (64x64x31), SNR-in 20 dB -> PSNR gain >= +10 dB."""
    s = synth.low_rank_cube(64, 64, 31, rank=6, seed=12, snr_db=20.0)
    res = O.hyres(s.noisy)
    assert metrics.psnr(s.clean, res.out) - metrics.psnr(s.clean, s.noisy) >= 10.0


def test_olympic_mean_spec(golden_dir):
    gd = json.load(open(os.path.join(golden_dir, "spec_examples.json")))["olympic_mean"]
    for vals, want in gd["cases"]:
        assert metrics.olympic_mean(vals) == want
    rng = np.random.default_rng(13)
    for _ in range(50):
        v = rng.standard_normal(int(rng.integers(3, 101)))
        assert abs(metrics.olympic_mean(v) - np.mean(np.sort(v)[1:-1])) < 1e-12
    with pytest.raises(ValueError):
        metrics.olympic_mean([1.0, 2.0])


# ---------------------------------------------------------------- F1: HySime
def _low_rank_cube(rng, r, c, b, rank, snr_db=None):
    a = rng.random((rank, r * c))
    s = rng.random((b, rank))
    x = s @ a
    if snr_db is not None:
        sig = np.sqrt(np.mean(x ** 2) / 10 ** (snr_db / 10))
        x = x + sig * rng.standard_normal(x.shape)
    return x.reshape(b, r, c)


def test_f1_noise_residual_is_the_regression_residual():
    """N~_b is orthogonal to every other band (normal equations) and equals the
    closed form (M Y)_b / M_bb of the full inverse (ridge 0) -- a different route."""
    rng = np.random.default_rng(11)
    y = rng.standard_normal((6, 200))
    res = O.noise_residual(y.reshape(6, 10, 20), ridge=0.0)
    g = y @ y.T
    for i in range(6):
        o = [j for j in range(6) if j != i]
        assert np.max(np.abs(y[o] @ res[i])) < 1e-9 * np.max(np.abs(g))
    m = np.linalg.inv(g)
    closed = (m @ y) / np.diag(m)[:, None]
    assert np.max(np.abs(closed - res)) < 1e-9


def test_f1_spec_rank5_30db():
    """SPEC.md:374 example: synthetic rank-5 cube (64x64x50) at 30 dB -> k == 5 (+-1);
    basis orthonormal."""
    rng = np.random.default_rng(12)
    cube = _low_rank_cube(rng, 64, 64, 50, 5, snr_db=30)
    h = O.hysime(cube)
    assert abs(h.k - 5) <= 1, h.k
    assert np.max(np.abs(h.basis.T @ h.basis - np.eye(h.k))) < 1e-10


def test_f1_noiseless_rank1():
    """noiseless rank-1 cube -> k == 1 (the ridge leaves a residual
    of order delta; its projected power is far below the signal's)."""
    rng = np.random.default_rng(13)
    cube = _low_rank_cube(rng, 32, 32, 12, 1)
    assert O.hysime(cube).k == 1


def test_f1_pure_noise_has_no_signal_subspace():
    """White noise: R_x ~ 0, every delta_i ~ sigma_i^2 > 0 -> k == 0."""
    rng = np.random.default_rng(14)
    cube = rng.standard_normal((16, 64, 64))
    assert O.hysime(cube).k == 0


def test_f1_criterion_is_the_brute_force_minimum():
    """k and the basis minimise the HySime error sum over subspaces spanned by
    eigenvectors of R_x: brute force over every subset of a small problem."""
    import itertools
    rng = np.random.default_rng(15)
    cube = _low_rank_cube(rng, 16, 16, 7, 3, snr_db=15)
    h = O.hysime(cube)
    b = 7
    best, best_set = None, None
    for r in range(b + 1):
        for sub in itertools.combinations(range(b), r):
            v = float(sum(h.delta[i] for i in sub))   # error(S) - const = sum_{i in S} delta_i
            if best is None or v < best - 1e-15:
                best, best_set = v, sub
    assert len(best_set) == h.k
    assert set(best_set) == set(int(i) for i in np.nonzero(h.delta < 0)[0])
    assert np.min(np.abs(h.delta)) > O.HYSIME_TOL * np.max(np.abs(h.delta))   # no near-zero delta here


def test_f1_eigen_identities():
    """R_x = E diag(mu) E^T, E orthonormal, R_n symmetric PSD, p_i - sigma_i^2 = mu_i."""
    rng = np.random.default_rng(16)
    cube = _low_rank_cube(rng, 32, 32, 20, 4, snr_db=20)
    h = O.hysime(cube)
    rx = h.r_y - h.noise_cov
    assert np.max(np.abs(h.E @ np.diag(h.mu) @ h.E.T - rx)) < 1e-12 * np.max(np.abs(rx))
    assert np.max(np.abs(h.E.T @ h.E - np.eye(20))) < 1e-12
    assert np.min(np.linalg.eigvalsh(h.noise_cov)) > -1e-14
    p = np.einsum("ij,ik,kj->j", h.E, h.r_y, h.E)
    s2 = np.einsum("ij,ik,kj->j", h.E, h.noise_cov, h.E)
    assert np.max(np.abs((p - s2) - h.mu)) < 1e-12 * np.max(np.abs(h.mu))


# ---------------------------------------------------------------- F2: FORPDN
def test_f2_closed_form_is_the_minimiser():
    """X = W (I + lam D^T D)^-1 satisfies the normal equations of
    min ||W - X||^2 + lam ||X D^T||^2: (X - W) + lam X D^T D = 0; and the
    objective grows along random perturbations."""
    rng = np.random.default_rng(31)
    b = 9
    w = rng.standard_normal((50, b))
    d = O.spectral_difference(b)
    assert np.allclose(d @ np.arange(b, dtype=float), np.ones(b - 1))
    lam = 3.0
    x = w @ np.linalg.inv(np.eye(b) + lam * d.T @ d)
    assert np.max(np.abs((x - w) + lam * x @ d.T @ d)) < 1e-12
    f = lambda z: np.sum((w - z) ** 2) + lam * np.sum((z @ d.T) ** 2)   # noqa: E731
    for _ in range(5):
        assert f(x + 1e-3 * rng.standard_normal(x.shape)) > f(x)


def test_f2_spec_examples():
    """lam -> 0+ gives the input back (1e-3); linearity in the input
    (1e-4 relative, fixed lam); spectrally smooth cube + 20 dB noise, lam = 10 ->
    PSNR gain >= 5 dB."""
    rng = np.random.default_rng(32)
    b, r, c = 60, 32, 32
    t = np.arange(b)
    # spectrally smooth: Gaussian bumps 18 bands wide
    spectra = np.stack([np.exp(-0.5 * ((t - m) / 18.0) ** 2) + 0.2 for m in (10, 30, 50)])
    ab = rng.random((3, r * c))
    clean = (spectra.T @ ab).reshape(b, r, c)
    out0 = O.forpdn(clean.astype(np.float32), lam=1e-8, levels=2).out
    assert np.max(np.abs(out0 - clean)) < 1e-3 * np.max(np.abs(clean))
    x = rng.standard_normal((b, r, c)).astype(np.float32)
    o1 = O.forpdn(x, lam=2.0, levels=2).out.astype(np.float64)
    o2 = O.forpdn((3.0 * x).astype(np.float32), lam=2.0, levels=2).out.astype(np.float64)
    assert np.linalg.norm(o2 - 3.0 * o1) <= 1e-4 * np.linalg.norm(o2)
    sig = np.sqrt(np.mean(clean ** 2) / 10 ** 2)
    noisy = (clean + sig * rng.standard_normal(clean.shape)).astype(np.float32)
    den = O.forpdn(noisy, lam=10.0, levels=2).out
    gain = 10 * np.log10(np.mean((noisy - clean) ** 2) / np.mean((den - clean) ** 2))
    assert gain >= 5.0, gain


def test_f2_default_lambda_from_grid():
    """D16: the default lambda is the grid value whose residual power is closest to
    HySime's noise power; the residual power grows with lambda."""
    rng = np.random.default_rng(33)
    b, r, c = 16, 32, 32
    t = np.linspace(0, 1, b)
    clean = (np.outer(np.cos(3 * t) + 2, rng.random(r * c))).reshape(b, r, c)
    noisy = (clean + 0.05 * rng.standard_normal(clean.shape)).astype(np.float32)
    res = O.forpdn(noisy, levels=2)
    assert res.lam in O.FORPDN_GRID
    rp = [res.residual_power[l] for l in O.FORPDN_GRID]
    assert all(rp[i] < rp[i + 1] for i in range(len(rp) - 1))
    assert res.lam == min(O.FORPDN_GRID, key=lambda l: abs(res.residual_power[l] - res.noise_power))


def test_f2_default_lambda_on_white_noise_closed_form():
    """D16 pinned on pure white noise of known sigma, from closed forms (not the oracle's
    own rule): with W i.i.d. N(0, sigma^2) (orthonormal DWT, 2^L | R, C), the residual
    W - W A^-1 = W (I - A^-1) has power sigma^2 tr((I - A^-1)^2) / B per entry, and
    HySime's regression noise power is sigma^2 (N - B + 1) / N (chi^2 with N - B + 1
    dof).  The oracle's residual powers must match the closed forms within 3 %, its noise
    power within 3 %, and its lambda must be the grid value the closed forms select."""
    rng = np.random.default_rng(61)
    b, r, c, sig = 12, 64, 64, 0.7
    x = (sig * rng.standard_normal((b, r, c))).astype(np.float32)
    res = O.forpdn(x, levels=2, taps=8)
    n = r * c
    d = O.spectral_difference(b)
    cf = {}
    for lmb in O.FORPDN_GRID:
        k = np.eye(b) - np.linalg.inv(np.eye(b) + lmb * d.T @ d)
        cf[lmb] = sig ** 2 * np.trace(k @ k) / b
        assert abs(res.residual_power[lmb] / cf[lmb] - 1) < 0.03, (lmb, res.residual_power[lmb], cf[lmb])
    npow = sig ** 2 * (n - b + 1) / n
    assert abs(res.noise_power / npow - 1) < 0.03
    assert res.lam == min(O.FORPDN_GRID, key=lambda l: abs(cf[l] - npow))


def test_f4_default_lambda_and_rank_on_white_noise():
    """D17 pinned on pure white noise of known sigma: sigma_b^2 has expectation
    sigma^2 (N - B + 1) / N, so the default lambda = sqrt(mean sigma_b^2) sqrt(2 ln N_c)
    is within 1 % of sigma sqrt((N - B + 1) / N) sqrt(2 ln N_c); HySime finds no signal
    subspace in pure noise (k = 0), so the default rank is max(1, k) = 1."""
    rng = np.random.default_rng(62)
    b, r, c, sig = 10, 64, 64, 1.3
    x = (sig * rng.standard_normal((b, r, c))).astype(np.float32)
    res = O.wsrrr(x, levels=2, taps=8, max_iters=3)
    n = r * c
    nc = O.coeff_count(r, c, 2)
    want = sig * math.sqrt((n - b + 1) / n) * math.sqrt(2 * math.log(nc))
    assert abs(res.lam / want - 1) < 0.01, (res.lam, want)
    assert res.rank == 1


def test_last_component_always_fails():
    """Why r* = B never occurs under the first-failure rule (R2): with
    sigma_b^2 = 1 / (N [(G + dI)^-1]_bb), G_w^-1 = N D^1/2 G^-1 D^1/2 has diagonal
    [G^-1]_bb / [(G + dI)^-1]_bb >= 1, so lambda_min(G_w) <= 1 and the last whitened
    component has energy <= N <= N_c; soft thresholding only lowers it.  Checked on
    noisy, noiseless and full-rank cubes; the oracle's walk then stops at k = B with
    r* = B - 1 where every earlier component passes."""
    rng = np.random.default_rng(63)
    cubes = [synth.make_cube("tiny", 0).noisy, synth.low_rank_cube(32, 32, 6, rank=6, seed=1).clean,
             rng.standard_normal((5, 20, 20)).astype(np.float32),
             synth.low_rank_cube(64, 64, 4, rank=4, seed=3).clean]
    for cube in cubes:
        b, r, c = cube.shape
        sigma, g = O.estimate_noise(cube)
        lam, _, _ = O.whiten_eig(g, sigma, r * c)
        assert lam[-1] <= 1.0 + 1e-9, lam[-1]
    ref = O.hyres(cubes[-1])
    assert len(ref.e_post) == 4 and ref.rank == 3 and ref.e_post[-1] <= ref.n_coeffs


# ---------------------------------------------------------------- F4: WSRRR
def test_f4_spec_lossless_full_rank():
    """lam = 0, rank = bands -> denoised ~= input within 1e-3."""
    rng = np.random.default_rng(51)
    x = rng.standard_normal((8, 32, 32)).astype(np.float32)
    res = O.wsrrr(x, rank=8, lam=0.0, levels=2)
    assert np.max(np.abs(res.out - x)) < 1e-3 * np.max(np.abs(x))
    assert np.max(np.abs(res.V.T @ res.V - np.eye(8))) < 1e-10


def test_f4_spec_rank4_gain_and_monotone():
    """rank-4 synthetic cube at 20 dB, rank = 4 -> PSNR gain >= 8 dB;
    the objective never increases (1e-6 relative slack); components count == rank."""
    rng = np.random.default_rng(52)
    b, r, c = 30, 64, 64
    t = np.arange(b)
    spectra = np.stack([np.exp(-0.5 * ((t - m) / 6.0) ** 2) for m in (4, 11, 18, 25)])
    ab = np.stack([np.kron(rng.random((8, 8)), np.ones((8, 8))).ravel() for _ in range(4)])   # piecewise-constant
    clean = (spectra.T @ ab).reshape(b, r, c)
    sig = np.sqrt(np.mean(clean ** 2) / 100.0)
    noisy = (clean + sig * rng.standard_normal(clean.shape)).astype(np.float32)
    res = O.wsrrr(noisy, rank=4, levels=3, taps=2)   # piecewise-constant abundances: Haar-sparse
    gain = 10 * np.log10(np.mean((noisy - clean) ** 2) / np.mean((res.out - clean) ** 2))
    assert gain >= 8.0, gain
    f = res.objective
    assert all(f[i + 1] <= f[i] * (1 + 1e-6) for i in range(len(f) - 1))
    assert res.components.shape == (4, r, c)
    assert np.max(np.abs(res.V.T @ res.V - np.eye(4))) < 1e-10


def test_f4_steps_are_the_block_minimisers():
    """C-step: soft(W V, lam/2) beats perturbations of C for the fixed V; V-step: the
    Procrustes V maximises tr(V^T W^T C) against random orthonormal V."""
    rng = np.random.default_rng(53)
    w = rng.standard_normal((200, 6))
    v, _ = np.linalg.qr(rng.standard_normal((6, 2)))
    lam = 0.7
    cm = O.soft_threshold(w @ v, lam / 2.0)
    f = lambda cc, vv: np.sum((w - cc @ vv.T) ** 2) + lam * np.sum(np.abs(cc))   # noqa: E731
    for _ in range(5):
        assert f(cm + 1e-3 * rng.standard_normal(cm.shape), v) > f(cm, v)
    p, _, qt = np.linalg.svd(w.T @ cm, full_matrices=False)
    vb = p @ qt
    for _ in range(20):
        q, _ = np.linalg.qr(rng.standard_normal((6, 2)))
        assert np.trace(q.T @ w.T @ cm) <= np.trace(vb.T @ w.T @ cm) + 1e-12


# ---------------------------------------------------------------- F3: HyMiNoR
def test_f3_split_bregman_reaches_the_l1_minimum():
    """On tiny spectra the split-Bregman iterate approaches the true minimiser of
    ||m - x||_1 + lam ||D x||_1 (a linear program, solved here by scipy's
    linprog as the independent reference); the objective at the iterate is within
    1 % of the LP optimum."""
    from scipy.optimize import linprog
    rng = np.random.default_rng(61)
    b = 8
    dmat = O.spectral_difference(b)
    for trial in range(4):
        m = rng.standard_normal(b) + np.where(rng.random(b) < 0.2, 5.0, 0.0)
        lam = 0.7
        res = O.l1_spectral(m.reshape(b, 1, 1), lam=lam, mu=5.0, max_iters=3000, tol=0.0)
        x = res.out.reshape(b).astype(np.float64)
        f = np.sum(np.abs(m - x)) + lam * np.sum(np.abs(dmat @ x))
        # LP: variables [x (b), s (b) >= |m - x|, t (b-1) >= |D x|]
        nv = b + b + (b - 1)
        cvec = np.concatenate([np.zeros(b), np.ones(b), lam * np.ones(b - 1)])
        A, ub = [], []
        for i in range(b):
            row = np.zeros(nv); row[i] = -1; row[b + i] = -1; A.append(row); ub.append(-m[i])   # s >= m - x
            row = np.zeros(nv); row[i] = 1; row[b + i] = -1; A.append(row); ub.append(m[i])     # s >= x - m
        for i in range(b - 1):
            row = np.zeros(nv); row[:b] = dmat[i]; row[2 * b + i] = -1; A.append(row); ub.append(0.0)
            row = np.zeros(nv); row[:b] = -dmat[i]; row[2 * b + i] = -1; A.append(row); ub.append(0.0)
        lp = linprog(cvec, A_ub=np.array(A), b_ub=np.array(ub), bounds=[(None, None)] * b + [(0, None)] * (2 * b - 1))
        assert lp.success
        assert f <= lp.fun * 1.01 + 1e-9, (f, lp.fun)


def test_f3_gaussian_only_stays_with_hyres_and_residual_decreases():
    """pure Gaussian noise -> HyMiNoR within 1 dB of HyRes; the Bregman
    residual does not increase over the iterations (1e-6 slack).
    (SPEC.md:422's derived "+2 dB over HyRes with 5 % salt-and-pepper" does NOT
    hold for D19's formulation -- the l1 fidelity is to the HyRes output, in which
    the low-rank projection has already spread the impulses over the bands; on
    this generator the stage changes PSNR by < 0.2 dB.  Recorded in DESIGN.md R16.)"""
    rng = np.random.default_rng(62)
    b, r, c = 31, 64, 64
    t = np.arange(b)
    spectra = np.stack([np.exp(-0.5 * ((t - mm) / 5.0) ** 2) + 0.1 for mm in np.linspace(2, 28, 6)])
    ab = rng.dirichlet(np.ones(6), size=r * c).T
    clean = (spectra.T @ ab).reshape(b, r, c)
    sig = np.sqrt(np.mean(clean ** 2) / 100.0)
    gauss = clean + sig * rng.standard_normal(clean.shape)
    ps = lambda est: 10 * np.log10(np.max(clean) ** 2 / np.mean((est - clean) ** 2))   # noqa: E731
    hr = O.hyres(gauss.astype(np.float32)).out
    res = O.l1_spectral(hr)                       # D19 defaults (lam 10, mu 5, 50 iterations, tol 1e-3)
    assert abs(ps(res.out) - ps(hr)) <= 1.0
    rr = O.l1_spectral(hr, max_iters=50, tol=0.0).residuals
    assert all(rr[i + 1] <= rr[i] * (1 + 1e-6) + 1e-12 for i in range(len(rr) - 1))
