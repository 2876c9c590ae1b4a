"""F4: WSRRR on the GPU (hyde_wsrrr) against the fp64 oracle
(oracle.wsrrr) on the same seeded cubes."""
import numpy as np
import pytest

from oracle import hyres_ref as O
from harness import metrics, synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def hy():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2204_06979_b200 as hy
    return hy


def _rank4(seed=52):
    rng = np.random.default_rng(seed)
    b, r, c = 30, 64, 64
    t = np.arange(b)
    spectra = np.stack([np.exp(-0.5 * ((t - m) / 6.0) ** 2) for m in (4, 11, 18, 25)])
    ab = np.stack([np.kron(rng.random((8, 8)), np.ones((8, 8))).ravel() for _ in range(4)])
    clean = (spectra.T @ ab).reshape(b, r, c)
    sig = np.sqrt(np.mean(clean ** 2) / 100.0)
    return clean, (clean + sig * rng.standard_normal(clean.shape)).astype(np.float32)


@pytest.mark.parametrize("taps", [2, 16])
def test_wsrrr_matches_oracle(hy, taps):
    clean, noisy = _rank4()
    ref = O.wsrrr(noisy, rank=4, levels=3, taps=taps)
    got = hy.wsrrr(torch.from_numpy(noisy).cuda(), rank=4, levels=3, taps=taps, components=True)
    assert abs(got["lam"] - ref.lam) <= 1e-6 * ref.lam
    f = got["objective"]
    assert all(f[i + 1] <= f[i] * (1 + 1e-6) for i in range(len(f) - 1))
    assert abs(f[-1] - ref.objective[-1]) <= 1e-4 * ref.objective[-1]
    out = got["out"].cpu().numpy()
    assert metrics.rel_l2(ref.out, out) <= 1e-4
    comps = got["components"].cpu().numpy()
    assert comps.shape == ref.components.shape
    # components are defined up to the sign of the columns of V (and C)
    for k in range(4):
        a, b_ = ref.components[k].ravel(), comps[k].ravel()
        s = np.sign(np.dot(a, b_)) or 1.0
        assert np.linalg.norm(s * b_ - a) <= 1e-3 * np.linalg.norm(a)


def test_wsrrr_default_rank_and_lambda(hy):
    s = synth.make_cube("tiny", 0)
    ref = O.wsrrr(s.noisy)
    got = hy.wsrrr(torch.from_numpy(s.noisy).cuda())
    assert got["rank"] == ref.rank
    assert abs(got["lam"] - ref.lam) <= 1e-4 * ref.lam
    assert metrics.rel_l2(ref.out, got["out"].cpu().numpy()) <= 1e-4


def test_wsrrr_lossless_full_rank(hy):
    rng = np.random.default_rng(51)
    x = rng.standard_normal((8, 32, 32)).astype(np.float32)
    got = hy.wsrrr(torch.from_numpy(x).cuda(), rank=8, lam=0.0, levels=2)["out"].cpu().numpy()
    assert np.max(np.abs(got - x)) < 1e-3 * np.max(np.abs(x))


def test_wsrrr_odd_shape_padded_levels(hy):
    """Odd extents (padded DWT levels: the coefficient Gram is taken over N_c != N),
    rank 3, fixed lambda, a few sweeps."""
    rng = np.random.default_rng(57)
    b, r, c = 19, 33, 45
    x = (rng.standard_normal((3, r * c)).T @ rng.random((3, b))).T.reshape(b, r, c)
    x = (x + 0.1 * rng.standard_normal(x.shape)).astype(np.float32)
    ref = O.wsrrr(x, rank=3, lam=0.2, levels=2, max_iters=6, tol=0.0)
    got = hy.wsrrr(torch.from_numpy(x).cuda(), rank=3, lam=0.2, levels=2, max_iters=6, tol=0.0)
    assert len(got["objective"]) == len(ref.objective) == 6
    assert metrics.rel_l2(ref.out, got["out"].cpu().numpy()) <= 1e-4
