"""F2: FORPDN on the GPU (hyde_forpdn) against the fp64 oracle
(oracle.forpdn): the same default lambda (D16) and the output to 1e-4 relative L2."""
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


@pytest.mark.parametrize("name", ["tiny", "small"])
def test_forpdn_default_lambda_matches_oracle(hy, name):
    s = synth.make_cube(name, 0)
    ref = O.forpdn(s.noisy)
    out, lam = hy.forpdn(torch.from_numpy(s.noisy).cuda(), return_lambda=True)
    assert lam == ref.lam, (lam, ref.lam, ref.residual_power, ref.noise_power)
    got = out.cpu().numpy()
    assert metrics.rel_l2(ref.out, got) <= 1e-4
    assert metrics.mpsnr(s.clean, got) > metrics.mpsnr(s.clean, s.noisy)


@pytest.mark.parametrize("lam", [0.1, 1.0, 37.5])
def test_forpdn_fixed_lambda_and_odd_shape(hy, lam):
    rng = np.random.default_rng(41)
    x = rng.standard_normal((13, 37, 50)).astype(np.float32)
    ref = O.forpdn(x, lam=lam, levels=1)
    got = hy.forpdn(torch.from_numpy(x).cuda(), lam=lam, levels=1).cpu().numpy()
    assert metrics.rel_l2(ref.out, got) <= 1e-5


def test_forpdn_in_place_and_errors(hy):
    s = synth.make_cube("tiny", 0)
    g = torch.from_numpy(s.noisy).cuda()
    a = hy.forpdn(g, lam=2.0).cpu().numpy()
    hy.forpdn(g, out=g, lam=2.0)
    assert np.array_equal(g.cpu().numpy(), a)
    with pytest.raises(hy.HydeError):
        hy.forpdn(g, lam=-1.0)
