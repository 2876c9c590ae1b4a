"""Stage-isolated parity: each CUDA stage, called through the C-ABI,
against the oracle's same stage on identical inputs."""
import math

import numpy as np
import pytest

from oracle import hyres_ref as O
from harness import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def hy():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2204_06979_b200 as hy
    return hy


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _quantized_gram(y, inv_s, c):
    """The Gram K1 defines (k_gram_tc.cu, DESIGN.md §4 K1), from the scales it chose:
    q = rint(y inv_s - c) (fp32 inv_s, the exact product, ties to even); a pixel with any
    value whose fma r = fp32(y inv_s + 2^23 + 32768 - c) leaves [2^23, 2^23 + 65535]
    is flagged and enters exactly (fp64 y y^T); every other pixel enters as
    s (q + c), s = 1 / inv_s, with the integer Gram exact:
    G = diag(s) [sum_unflagged (q + c)(q + c)^T] diag(s) + sum_flagged y y^T."""
    y = np.asarray(y, dtype=np.float32)
    isl = inv_s.astype(np.longdouble)
    # the kernel's rounding exactly: r = fp32(y inv_s + kf), kf = 2^23 + 32768 - c
    # (one fma), in range iff 2^23 <= r <= 2^23 + 65535; just below 2^23 the fp32
    # spacing is 1/2, so y inv_s - c in (-32768.5, -32768.25) is flagged although
    # rint() would give -32768
    kf = (8421376 - c.astype(np.int64)).astype(np.longdouble)
    r = (y.astype(np.longdouble) * isl[:, None] + kf[:, None]).astype(np.float32).astype(np.float64)
    flag = ((r < 8388608.0) | (r > 8388608.0 + 65535.0)).any(axis=0)
    q = np.rint(y.astype(np.longdouble) * isl[:, None] - c[:, None].astype(np.longdouble))
    qc = (q[:, ~flag].astype(np.int64) + c[:, None])
    assert float(np.max(np.abs(qc))) ** 2 * qc.shape[1] < 2.0 ** 62
    t = qc @ qc.T
    s = 1.0 / inv_s.astype(np.float64)
    yf = y[:, flag].astype(np.float64)
    return (t.astype(np.float64) * s[:, None]) * s[None, :] + yf @ yf.T, int(flag.sum())


def _rounding_bound(y, inv_s):
    """Rigorous bound on |G_K1 - Y Y^T| from the rounding alone: each unflagged value
    moves by |e| <= s/2 (s = 1 / inv_s), so |sum_p y_i y_j - yh_i yh_j| <=
    s_j/2 sum|y_i| + s_i/2 sum|y_j| + N s_i s_j / 4 (flagged pixels are exact)."""
    y = np.asarray(y, dtype=np.float64)
    s = 1.0 / inv_s.astype(np.float64)
    a = np.sum(np.abs(y), axis=1)
    return 0.5 * (np.outer(a, s) + np.outer(s, a)) + 0.25 * y.shape[1] * np.outer(s, s)


@pytest.mark.parametrize("name", ["tiny", "small", "medium"])
def test_gram_matches_oracle(hy, name):
    """Tensor-core Gram vs the fp64 oracle: only the 16-bit centred rounding of the
    unflagged values remains (<1e-6 relative; the medium cube's impulse noise is flagged
    or inside the robust range).  Was 1e-5 with the max-scaled 15-bit grid; every element
    must also sit inside the rigorous rounding bound of the scales K1 chose."""
    s = synth.make_cube(name, 0)
    x = dev(s.noisy)
    g = hy.stages.gram(x).cpu().numpy()
    ref = O.gram(s.noisy)
    assert np.max(np.abs(g - ref)) / np.max(np.abs(ref)) < 5e-6
    inv_s, _, _ = hy.stages.gram_quant(x)
    assert np.all(np.abs(g - ref) <= _rounding_bound(s.noisy.reshape(s.noisy.shape[0], -1), inv_s)
                  + 1e-13 * np.max(np.abs(ref)))
    assert np.array_equal(g, g.T)
    assert np.min(np.linalg.eigvalsh(g)) > -1e-9 * np.max(np.abs(g))


@pytest.mark.parametrize("name", ["tiny", "small", "medium"])
def test_gram_is_exact_integer_gram(hy, name):
    """The int8 tcgen05 products and the flagged-pixel fix are exact: GPU G equals the
    Gram of the quantised cube with the flagged pixels exact."""
    s = synth.make_cube(name, 0)
    b = s.noisy.shape[0]
    x = dev(s.noisy)
    g = hy.stages.gram(x).cpu().numpy()
    inv_s, c, nflag = hy.stages.gram_quant(x)
    ref, nref = _quantized_gram(s.noisy.reshape(b, -1), inv_s, c)
    assert nflag == nref
    assert np.max(np.abs(g - ref)) / np.max(np.abs(ref)) < 1e-14


def test_gram_ragged_and_tiny_shapes(hy):
    rng = np.random.default_rng(0)
    for b, n in [(3, 5), (7, 1000), (65, 333), (129, 4097), (160, 2049), (224, 70001), (200, 31), (256, 2049),
                 (224, 131075)]:
        y = rng.standard_normal((b, n)).astype(np.float32)
        y[rng.random(y.shape) < 0.01] *= 30.0          # heavy tails
        y[:, 2] = 0.0                                   # a dead pixel
        x = dev(y.reshape(b, n, 1))
        g = hy.stages.gram(x).cpu().numpy()
        ref = y.astype(np.float64) @ y.astype(np.float64).T
        if b <= 224:   # tensor-core path: exact Gram of the quantised cube, outliers exact
            inv_s, c, nflag = hy.stages.gram_quant(x)
            q, nref = _quantized_gram(y, inv_s, c)
            assert nflag == nref, (b, n, nflag, nref)
            assert np.max(np.abs(g - q)) / np.max(np.abs(ref)) < 1e-14, (b, n)
            assert np.all(np.abs(g - ref) <= _rounding_bound(y, inv_s) + 1e-13 * np.max(np.abs(ref))), (b, n)
            if n >= 1000:   # averaging over pixels; a 5-pixel band keeps its 16-bit rounding
                # 1 % of values x 30 land in most sample blocks and widen R (the bound above still holds)
                assert np.max(np.abs(g - ref)) / np.max(np.abs(ref)) < 5e-5, (b, n)
        else:          # fp64 SIMT fallback
            assert np.max(np.abs(g - ref)) / np.max(np.abs(ref)) < 1e-13, (b, n)


@pytest.mark.parametrize("mult", [10.0, 30.0, 100.0, 1000.0, 1e6])
def test_gram_outlier_pixels_exact(hy, mult):
    """A hot pixel at mult x the band RMS in every band, a 1e3 x spike in one band, a
    saturated row and a dead band: the flagged pixels enter exactly, so the Gram stays
    ~1e-8 from fp64 whatever the dynamic range (reduced precision on
    extreme scales)."""
    s = synth.make_cube("small", 0)
    cube = s.noisy.copy()
    b = cube.shape[0]
    rms = np.sqrt(np.mean(cube.reshape(b, -1).astype(np.float64) ** 2, axis=1))
    cube[:, 70, 70] = (mult * rms).astype(np.float32)
    cube[50, 10, 20] = np.float32(1e3 * rms[50])
    cube[7, 100, :] = np.float32(cube[7].max() * 4)
    cube[120] = 0.0
    x = dev(cube)
    g = hy.stages.gram(x).cpu().numpy()
    ref = O.gram(cube)
    inv_s, c, nflag = hy.stages.gram_quant(x)
    q, nref = _quantized_gram(cube.reshape(b, -1), inv_s, c)
    assert nflag == nref and nflag >= 2
    assert np.max(np.abs(g - q)) / np.max(np.abs(ref)) < 1e-14
    # the outliers are exact: the error is the plain cube's rounding, inside its bound
    assert np.all(np.abs(g - ref) <= _rounding_bound(cube.reshape(b, -1), inv_s) + 1e-13 * np.max(np.abs(ref)))
    d = np.abs(g - ref) / np.sqrt(np.outer(np.diag(ref), np.diag(ref)) + 1e-300)
    assert np.max(d[np.ix_(np.arange(b) != 120, np.arange(b) != 120)]) < 1e-6
    assert np.all(g[120] == 0.0)


@pytest.mark.parametrize("name", ["tiny", "small", "medium", "wide"])
def test_noise_and_eig_match_oracle(hy, name):
    s = synth.make_cube(name, 0)
    b, r, c = s.noisy.shape
    n = r * c
    g = O.gram(s.noisy)
    sig_ref, _ = O.estimate_noise(s.noisy)
    lam_ref, v_ref, _ = O.whiten_eig(g, sig_ref, n)
    k = min(16, b)
    sig, lam, V = hy.stages.eig(dev(g), n, k)
    sig, lam, V = sig.cpu().numpy(), lam.cpu().numpy(), V.cpu().numpy()
    assert np.max(np.abs(sig / sig_ref - 1)) < 1e-9
    assert np.max(np.abs(lam - lam_ref)) < 1e-11 * lam_ref[0]
    # eigenvectors: compare where the eigenvalue is separated from its neighbours
    for j in range(k):
        gap = min([abs(lam_ref[j] - lam_ref[i]) for i in range(b) if i != j])
        if gap > 1e-6 * lam_ref[0]:
            err = np.max(np.abs(V[:, j] - v_ref[:, j]))
            assert err < 1e-16 * lam_ref[0] / gap * 1e3 + 1e-10, (j, err, gap)
    assert np.max(np.abs(V.T @ V - np.eye(k))) < 1e-8


@pytest.mark.parametrize("b,r,c,kmax", [(3, 17, 33, 16), (4, 20, 20, 16), (6, 20, 20, 16), (9, 31, 29, 16),
                                        (33, 40, 40, 16), (224, 40, 40, 16), (129, 30, 30, 32), (256, 50, 50, 32)])
def test_eigenpairs_are_eigenpairs(hy, b, r, c, kmax):
    """Every returned pair satisfies G_w v = lam v and V is orthonormal (small and odd band counts,
    the tridiagonal edge cases, B = 256 -- every row slot of the 16-CTA cluster -- and 32
    eigenpairs, two per CTA), independent of how close the eigenvalues are."""
    s = synth.low_rank_cube(r, c, b, rank=min(3, b - 1), seed=b, snr_db=20.0)
    n = r * c
    g = O.gram(s.noisy)
    sig_ref, _ = O.estimate_noise(s.noisy)
    k = min(kmax, b)
    sig, lam, V = hy.stages.eig(dev(g), n, k)
    sig, lam, V = sig.cpu().numpy(), lam.cpu().numpy(), V.cpu().numpy()
    assert np.max(np.abs(sig / sig_ref - 1)) < 1e-9
    gw = g / np.outer(sig, sig) / n
    lam_ref = np.sort(np.linalg.eigvalsh(gw))[::-1]
    assert np.max(np.abs(lam - lam_ref)) < 1e-11 * lam_ref[0]
    assert np.max(np.abs(gw @ V - V * lam[None, :k])) < 1e-9 * lam_ref[0]
    assert np.max(np.abs(V.T @ V - np.eye(k))) < 1e-8
    for j in range(k):                      # sign convention (S:181 D6)
        i = int(np.argmax(np.abs(V[:, j])))
        assert V[i, j] > 0


@pytest.mark.parametrize("name", ["tiny", "small", "medium", "wide"])
def test_lanczos_first_chunk_matches_oracle(hy, name):
    """The hot path's first chunk (K2 phase 2L: Lanczos on G_w - I, hyde_k_eig without
    eigenvalues, K = 4): every pair is an eigenpair of G_w, its Rayleigh quotient is the
    oracle's eigenvalue, the vectors match the oracle's (D6 signs) where the eigenvalue is
    separated from its neighbours, and they are orthonormal."""
    s = synth.make_cube(name, 0)
    b, r, c = s.noisy.shape
    n = r * c
    g = O.gram(s.noisy)
    sig_ref, _ = O.estimate_noise(s.noisy)
    lam_ref, v_ref, gw = O.whiten_eig(g, sig_ref, n)
    k = 4
    sig, lam, V = hy.stages.eig(dev(g), n, k, all_lam=False)
    assert lam is None
    sig, V = sig.cpu().numpy(), V.cpu().numpy()
    assert np.max(np.abs(sig / sig_ref - 1)) < 1e-9
    gw = g / np.outer(sig, sig) / n
    rq = np.einsum("ij,ij->j", V, gw @ V)
    assert np.max(np.abs(rq - lam_ref[:k])) < 1e-11 * lam_ref[0]
    assert np.max(np.abs(gw @ V - V * rq[None, :])) < 1e-9 * lam_ref[0]
    assert np.max(np.abs(V.T @ V - np.eye(k))) < 1e-10
    for j in range(k):
        gap = min([abs(lam_ref[j] - lam_ref[i]) for i in range(b) if i != j])
        if gap > 1e-6 * lam_ref[0]:
            err = np.max(np.abs(V[:, j] - v_ref[:, j]))
            assert err < 1e-12 * lam_ref[0] / gap + 1e-10, (j, err, gap)


def test_estimate_noise_api(hy):
    s = synth.make_cube("small", 0)
    sig, g, res = hy.estimate_noise(dev(s.noisy), return_gram=True, return_residual=True)
    sig_ref, g_ref, res_ref = O.estimate_noise(s.noisy, want_residual=True)
    # sigma within 1e-5 (the 16-bit centred rounding, DESIGN.md §4 K1)
    assert np.max(np.abs(sig.cpu().numpy() / sig_ref - 1)) < 1e-5
    assert np.max(np.abs(g.cpu().numpy() - g_ref)) / np.max(np.abs(g_ref)) < 1e-6
    rr = res.cpu().numpy().astype(np.float64)
    assert np.linalg.norm(rr - res_ref) / np.linalg.norm(res_ref) < 1e-4


def test_project_matches_fp64(hy):
    rng = np.random.default_rng(1)
    for b, n, k in [(32, 4096, 16), (200, 21025, 16), (7, 1001, 3), (103, 207400, 32), (50, 4099, 9)]:
        y = rng.standard_normal((b, n)).astype(np.float32)
        w = rng.standard_normal((b, k)).astype(np.float32)
        e = hy.stages.project(dev(y.reshape(b, n, 1)), dev(w)).cpu().numpy()
        ref = w.astype(np.float64).T @ y.astype(np.float64)
        assert np.max(np.abs(e - ref)) / np.max(np.abs(ref)) < 2e-6, (b, n, k)


DWT_SHAPES = [(64, 64, 2), (145, 145, 3), (610, 340, 4), (349, 1905, 4), (37, 50, 1), (17, 33, 2), (256, 256, 4)]


@pytest.mark.parametrize("taps", [2, 8, 16])
@pytest.mark.parametrize("shape", DWT_SHAPES)
def test_dwt_forward_and_inverse_match_oracle(hy, taps, shape):
    r, c, lv = shape
    rng = np.random.default_rng(2)
    x = rng.standard_normal((2, r, c)).astype(np.float32)
    co = hy.stages.dwt_fwd(dev(x), lv, taps).cpu().numpy()
    for i in range(2):
        ref = np.concatenate([s.ravel() for s in O.flatten_coeffs(O.dwt2(x[i], lv, taps))])
        assert co.shape[1] == ref.size
        assert np.max(np.abs(co[i] - ref)) < 2e-5 * max(1.0, np.max(np.abs(ref)))
    back = hy.stages.idwt(dev(co), r, c, lv, taps).cpu().numpy()
    assert np.max(np.abs(back - x)) < 5e-5
    # inverse of arbitrary coefficients vs the oracle's adjoint synthesis
    cr = rng.standard_normal(co.shape).astype(np.float32)
    img = hy.stages.idwt(dev(cr), r, c, lv, taps).cpu().numpy()
    tmpl = O.dwt2(np.zeros((r, c)), lv, taps)
    sizes = [s.size for s in O.flatten_coeffs(tmpl)]
    offs = np.cumsum([0] + sizes)
    for i in range(2):
        subs = [cr[i, offs[j]:offs[j + 1]].reshape(O.flatten_coeffs(tmpl)[j].shape) for j in range(len(sizes))]
        ref = O.idwt2(O.unflatten_coeffs([sb.astype(np.float64) for sb in subs], tmpl), taps)
        assert np.max(np.abs(img[i] - ref)) < 5e-5 * max(1.0, np.max(np.abs(ref)))


def _oracle_sure_on(co_row, r, c, lv):
    tmpl = O.dwt2(np.zeros((r, c)), lv, 16)
    subs = O.flatten_coeffs(tmpl)
    offs = np.cumsum([0] + [s.size for s in subs])
    out = []
    for j in range(len(subs)):
        out.append(O.sure_threshold(co_row[offs[j]:offs[j + 1]].astype(np.float64)))
    return out, offs


@pytest.mark.parametrize("shape", [(64, 64, 2), (145, 145, 3), (1024, 1024, 5), (349, 1905, 4)])
def test_sure_indices_bit_exact(hy, shape):
    r, c, lv = shape
    rng = np.random.default_rng(3)
    nc = O.coeff_count(r, c, lv)
    rows = []
    # sparse signal + unit noise; pure noise; heavy signal
    a = rng.standard_normal(nc); a[rng.random(nc) < 0.05] *= 20
    rows.append(a)
    rows.append(rng.standard_normal(nc))
    b = rng.standard_normal(nc) * 0.3; b[rng.random(nc) < 0.3] += 50
    rows.append(b)
    co = np.stack(rows).astype(np.float32)
    g = dev(co)
    ks, ts, ep = hy.stages.sure(g, r, c, lv)
    ks, ts, ep, soft = ks.cpu().numpy(), ts.cpu().numpy(), ep.cpu().numpy(), g.cpu().numpy()
    for i in range(co.shape[0]):
        res, offs = _oracle_sure_on(co[i], r, c, lv)
        e_ref = 0.0
        for j, sr in enumerate(res):
            scale = offs[j + 1] - offs[j] + float(np.sum(co[i, offs[j]:offs[j + 1]].astype(np.float64) ** 2))
            if sr.margin > 1e-9 * scale:
                assert ks[i, j] == sr.k, (i, j, ks[i, j], sr.k, sr.margin)
                assert ts[i, j] == np.float32(sr.t)
            st = O.soft_threshold(co[i, offs[j]:offs[j + 1]].astype(np.float64), float(ts[i, j]))
            assert np.max(np.abs(soft[i, offs[j]:offs[j + 1]] - st)) < 1e-5 * max(1.0, float(ts[i, j]))
            e_ref += float(np.sum(st ** 2))
        assert abs(ep[i] - e_ref) <= 1e-6 * max(1.0, e_ref)


def test_sure_many_subbands_single_cta_path(hy):
    """Enough big subbands in one launch that each takes ONE CTA (no cluster split):
    same exact indices as the oracle."""
    r, c, lv = 1024, 1024, 5
    nc = O.coeff_count(r, c, lv)
    rng = np.random.default_rng(7)
    rows = []
    for i in range(20):
        a = rng.standard_normal(nc) * (1.0 + 0.1 * i)
        a[rng.random(nc) < 0.02 * (i % 5)] *= 15
        rows.append(a)
    co = np.stack(rows).astype(np.float32)
    g = dev(co)
    ks, ts, ep = hy.stages.sure(g, r, c, lv)
    ks, ts, ep = ks.cpu().numpy(), ts.cpu().numpy(), ep.cpu().numpy()
    for i in range(co.shape[0]):
        res, offs = _oracle_sure_on(co[i], r, c, lv)
        e_ref = 0.0
        for j, sr in enumerate(res):
            x = co[i, offs[j]:offs[j + 1]].astype(np.float64)
            scale = x.size + float(np.sum(x ** 2))
            if sr.margin > 1e-9 * scale:
                assert ks[i, j] == sr.k and ts[i, j] == np.float32(sr.t), (i, j, ks[i, j], sr.k)
            e_ref += float(np.sum(O.soft_threshold(x, float(ts[i, j])) ** 2))
        assert abs(ep[i] - e_ref) <= 1e-6 * max(1.0, e_ref)


def test_sure_edge_cases(hy):
    r, c, lv = 64, 64, 2
    nc = O.coeff_count(r, c, lv)
    rng = np.random.default_rng(4)
    cases = [np.zeros(nc), np.full(nc, 0.5), np.full(nc, 7.0),
             np.round(rng.standard_normal(nc) * 4) / 4,                  # many exact duplicates
             np.where(rng.random(nc) < 0.5, 0.0, rng.standard_normal(nc))]
    co = np.stack(cases).astype(np.float32)
    ks, ts, ep = hy.stages.sure(dev(co), r, c, lv)
    ks, ts = ks.cpu().numpy(), ts.cpu().numpy()
    for i in range(co.shape[0]):
        res, offs = _oracle_sure_on(co[i], r, c, lv)
        for j, sr in enumerate(res):
            scale = offs[j + 1] - offs[j] + float(np.sum(co[i, offs[j]:offs[j + 1]].astype(np.float64) ** 2))
            if sr.margin > 1e-9 * scale:
                assert ks[i, j] == sr.k and ts[i, j] == np.float32(sr.t), (i, j, ks[i, j], sr.k)


def test_sure_catch_all_bin_edges(hy):
    """Keys at the edges of the first histogram pass's binned range [2^-40, 2^24): values
    in [2^24, 2^24 (1 + 1/64)) -- the first bin width past the range -- belong to the
    high catch-all bin, values just under 2^-40 to the low one; both in big subbands (the
    histogram path, n > 8192) and mixed with unit noise.  k* / t* bit-exact vs the
    oracle's exact SURE, E_post to 1e-12."""
    r, c, lv = 256, 256, 1
    nc = O.coeff_count(r, c, lv)
    rng = np.random.default_rng(9)
    rows = []
    for big in (2.0 ** 24, 2.0 ** 24 * 1.01, 2.0 ** 24 * (1 + 1 / 64), 3.0e7):
        a = rng.standard_normal(nc)
        idx = rng.choice(nc, 40, replace=False)
        a[idx[:20]] = big * (1 + 1e-3 * rng.random(20)) * np.sign(rng.standard_normal(20))
        a[idx[20:]] = 2.0 ** -41 * (1 + rng.random(20))
        rows.append(a)
    co = np.stack(rows).astype(np.float32)
    g = dev(co)
    ks, ts, ep = hy.stages.sure(g, r, c, lv)
    ks, ts, ep = ks.cpu().numpy(), ts.cpu().numpy(), ep.cpu().numpy()
    for i in range(co.shape[0]):
        res, offs = _oracle_sure_on(co[i], r, c, lv)
        e_ref = 0.0
        for j, sr in enumerate(res):
            scale = offs[j + 1] - offs[j] + float(np.sum(co[i, offs[j]:offs[j + 1]].astype(np.float64) ** 2))
            if sr.margin > 1e-9 * scale:
                assert ks[i, j] == sr.k and ts[i, j] == np.float32(sr.t), (i, j, ks[i, j], sr.k)
            e_ref += float(np.sum(O.soft_threshold(co[i, offs[j]:offs[j + 1]].astype(np.float64), float(ts[i, j])) ** 2))
        assert abs(ep[i] - e_ref) <= 1e-12 * e_ref, (i, ep[i], e_ref)


def test_reconstruct_matches_fp64(hy):
    rng = np.random.default_rng(5)
    for b, n, r in [(224, 4096, 1), (32, 1001, 3), (200, 21025, 9), (17, 64, 17)]:
        e = rng.standard_normal((r, n)).astype(np.float32)
        u = rng.standard_normal((b, r)).astype(np.float32)
        out = hy.stages.reconstruct(dev(e), dev(u)).cpu().numpy()
        ref = u.astype(np.float64) @ e.astype(np.float64)
        assert np.max(np.abs(out - ref)) / np.max(np.abs(ref)) < 1e-6


@pytest.mark.parametrize("shape", [(64, 64, 2), (145, 145, 3), (256, 256, 4), (37, 50, 1)])
def test_wavelet_shrink_matches_oracle(hy, shape):
    """hyde_wavelet_shrink (A4 -> A5 -> A6a as the hot path runs them) vs the oracle's
    dwt2 -> per-subband SURE -> soft threshold -> idwt2 on the same images."""
    r, c, lv = shape
    rng = np.random.default_rng(6)
    yy, xx = np.mgrid[0:r, 0:c]
    imgs = []
    for k in range(3):
        clean = (8.0 / (k + 1)) * np.sin(xx / (5.0 + 3 * k)) * np.cos(yy / (7.0 + k))
        imgs.append(clean + rng.standard_normal((r, c)))
    x = np.stack(imgs).astype(np.float32)
    out, ks, ts, ep = hy.stages.wavelet_shrink(dev(x), lv)
    out, ks, ts, ep = out.cpu().numpy(), ks.cpu().numpy(), ts.cpu().numpy(), ep.cpu().numpy()
    co = hy.stages.dwt_fwd(dev(x), lv).cpu().numpy()          # the coefficients SURE saw
    for i in range(x.shape[0]):
        res, offs = _oracle_sure_on(co[i], r, c, lv)
        for j, sr in enumerate(res):
            scale = offs[j + 1] - offs[j] + float(np.sum(co[i, offs[j]:offs[j + 1]].astype(np.float64) ** 2))
            if sr.margin > 1e-9 * scale:
                assert ks[i, j] == sr.k and ts[i, j] == np.float32(sr.t), (i, j, ks[i, j], sr.k)
        subs = O.flatten_coeffs(O.dwt2(x[i].astype(np.float64), lv, 16))
        soft = [O.soft_threshold(sb, float(ts[i, j])) for j, sb in enumerate(subs)]
        tmpl = O.dwt2(np.zeros((r, c)), lv, 16)
        ref = O.idwt2(O.unflatten_coeffs(soft, tmpl), 16)
        assert np.linalg.norm(out[i] - ref) <= 1e-4 * np.linalg.norm(ref)
        e_ref = sum(float(np.sum(sb ** 2)) for sb in soft)
        assert abs(ep[i] - e_ref) <= 1e-5 * e_ref
    # in place (out == images) gives the same result
    g = dev(x)
    same = hy.stages.wavelet_shrink(g, lv, out=g, stats=False)
    assert np.array_equal(same.cpu().numpy(), out)


def test_wavelet_shrink_analysis_only(hy):
    """out == NULL runs DWT + SURE only (the bench's DWT+SURE wall time): the same
    thresholds and k* as the full call, on 70 images with a ragged shape."""
    rng = np.random.default_rng(8)
    r, c, lv, cnt = 64, 96, 2, 70
    yy, xx = np.mgrid[0:r, 0:c]
    x = np.stack([(6.0 / (1 + k % 5)) * np.sin(xx / (4.0 + k % 7)) * np.cos(yy / (6.0 + k % 3))
                  + rng.standard_normal((r, c)) for k in range(cnt)]).astype(np.float32)
    _, k1, t1, e1 = hy.stages.wavelet_shrink(dev(x), lv)
    _, ka, ta, ea = hy.stages.wavelet_shrink(dev(x), lv, analyze_only=True)
    assert np.array_equal(ka.cpu().numpy(), k1.cpu().numpy())
    assert np.array_equal(ta.cpu().numpy(), t1.cpu().numpy())
    assert np.array_equal(ea.cpu().numpy(), e1.cpu().numpy())


def test_sure_dense_window_refinement(hy):
    """Subbands whose first-pass window exceeds the 8192-key capacity (a dense cluster
    of magnitudes where SURE is flat) go through the finer re-binning passes and still
    give the oracle's exact index; a subband with only a few distinct values (runs)
    takes the closed form."""
    r, c, lv = 1024, 1024, 5
    nc = O.coeff_count(r, c, lv)
    rng = np.random.default_rng(8)
    rows = []
    a = rng.standard_normal(nc)
    a[:nc // 3] = rng.uniform(3.4, 3.7, nc // 3) * np.sign(rng.standard_normal(nc // 3))
    rows.append(a)
    b = rng.standard_normal(nc)
    idx = rng.random(nc) < 0.15
    b[idx] = 2.5 + 1e-3 * rng.standard_normal(int(idx.sum()))
    rows.append(b)
    d = np.round(rng.standard_normal(nc) * 2) / 2          # runs of equal magnitudes
    rows.append(d)
    co = np.stack(rows).astype(np.float32)
    ks, ts, ep = hy.stages.sure(dev(co), r, c, lv)
    ks, ts, ep = ks.cpu().numpy(), ts.cpu().numpy(), ep.cpu().numpy()
    for i in range(co.shape[0]):
        res, offs = _oracle_sure_on(co[i], r, c, lv)
        e_ref = 0.0
        for j, sr in enumerate(res):
            x = co[i, offs[j]:offs[j + 1]].astype(np.float64)
            if sr.margin > 1e-9 * (x.size + float(np.sum(x ** 2))):
                assert ks[i, j] == sr.k and ts[i, j] == np.float32(sr.t), (i, j, ks[i, j], sr.k)
            e_ref += float(np.sum(O.soft_threshold(x, float(ts[i, j])) ** 2))
        assert abs(ep[i] - e_ref) <= 1e-6 * max(1.0, e_ref)
