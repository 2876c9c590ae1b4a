"""F1: HySime on the GPU (hyde_hysime) against the fp64 oracle
(oracle.hysime) on the same seeded cubes: identical k, the noise covariance, the
delta criterion and the selected basis."""
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


def _low_rank(rng, r, c, b, rank, snr_db):
    a = rng.random((rank, r * c))
    s = rng.random((b, rank))
    x = s @ a
    sig = np.sqrt(np.mean(x ** 2) / 10 ** (snr_db / 10))
    return (x + sig * rng.standard_normal(x.shape)).reshape(b, r, c).astype(np.float32)


CASES = [("lowrank5", None), ("tiny", None), ("small", None), ("medium", None)]


def _cube(name):
    if name == "lowrank5":
        return _low_rank(np.random.default_rng(21), 64, 64, 50, 5, 30)
    return synth.make_cube(name, 0).noisy


@pytest.mark.parametrize("name", [c[0] for c in CASES])
def test_hysime_matches_oracle(hy, name):
    cube = _cube(name)
    ref = O.hysime(cube)
    got = hy.hysime(torch.from_numpy(np.ascontiguousarray(cube)).cuda())
    assert got["k"] == ref.k, (got["k"], ref.k)
    nc = got["noise_cov"].cpu().numpy()
    # the GPU Gram is the exact Gram of a 15-bit quantisation (DESIGN.md §4 K1)
    assert np.max(np.abs(nc - ref.noise_cov)) <= 1e-4 * np.max(np.abs(np.diag(ref.noise_cov)))
    mu = got["mu"].cpu().numpy()
    assert np.max(np.abs(mu - ref.mu)) <= 1e-5 * np.max(np.abs(ref.mu))
    d = got["delta"].cpu().numpy()
    scale = np.max(np.abs(ref.delta))
    # delta of the signal components (well-separated eigenvalues) to 1e-5
    sel = np.arange(ref.k)
    assert np.max(np.abs(d[sel] - ref.delta[sel])) <= 1e-5 * scale if ref.k else True
    bas = got["basis"].cpu().numpy()
    assert bas.shape == ref.basis.shape
    if ref.k:
        assert np.max(np.abs(bas - ref.basis)) < 1e-4
        assert np.max(np.abs(bas.T @ bas - np.eye(ref.k))) < 1e-9


def test_hysime_noiseless_rank1(hy):
    rng = np.random.default_rng(13)
    a = rng.random((1, 32 * 32))
    s = rng.random((12, 1))
    cube = (s @ a).reshape(12, 32, 32).astype(np.float32)
    assert hy.hysime(torch.from_numpy(cube).cuda())["k"] == O.hysime(cube).k == 1
