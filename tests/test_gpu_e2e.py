"""End-to-end parity of the CUDA HyRes path (through the C-ABI) with the fp64 oracle
(SURVEY.md §4 T2/T3): relative L2 <= 1e-4, |dMPSNR| <= 0.01 dB, identical rank r*
(north_star acceptance), plus invariances, edge cases and error paths."""
import numpy as np
import pytest

from oracle import hyres_ref as O
from harness import synth, metrics

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

REL_L2 = 1e-4
DMPSNR = 0.01


@pytest.fixture(scope="module")
def hy():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2204_06979_b200 as hy
    return hy


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _compare(s, ref, out, info):
    assert info["rank"] == ref.rank
    assert info["levels"] == ref.levels
    assert info["n_coeffs"] == ref.n_coeffs
    assert metrics.rel_l2(ref.out, out) <= REL_L2
    assert abs(metrics.mpsnr(s.clean, out) - metrics.mpsnr(s.clean, ref.out)) <= DMPSNR


@pytest.mark.parametrize("name", ["tiny", "small", "medium", "wide"])
def test_hyres_matches_oracle(hy, name):
    s = synth.make_cube(name, 0)
    ref = O.hyres(s.noisy)
    out, info = hy.hyres(dev(s.noisy), return_info=True)
    _compare(s, ref, out.cpu().numpy(), info)


@pytest.mark.slow
def test_hyres_large_matches_oracle(hy):
    s = synth.make_cube("large", 0)
    ref = O.hyres(s.noisy)
    out, info = hy.hyres(dev(s.noisy), return_info=True)
    _compare(s, ref, out.cpu().numpy(), info)


def test_batched_lanes_reuse_and_mixed_cubes(hy):
    """More cubes than the batched path's 8 lanes (lanes reused, cube i on lane
    i % 8), mixed contents: each output equals the single-cube result, bit for bit."""
    cubes = [synth.make_cube("tiny", sd).noisy for sd in range(11)]
    cubes[5] = synth.low_rank_cube(64, 64, 32, rank=4, seed=5).clean     # a noiseless one in the middle
    x = dev(np.stack(cubes))
    outs, infos = hy.hyres_batched(x, return_info=True)
    for i in range(len(cubes)):
        single, info = hy.hyres(x[i].contiguous(), return_info=True)
        assert torch.equal(single, outs[i]), i
        assert infos[i]["rank"] == info["rank"]


def test_batched_matches_single_and_oracle(hy):
    cfg = synth.CONFIGS["batched"]
    seeds = [0, 1, 2]
    samples = [synth.make_cube(cfg, sd) for sd in seeds]
    cubes = dev(np.stack([x.noisy for x in samples]))
    outs, infos = hy.hyres_batched(cubes, return_info=True)
    for i, s in enumerate(samples):
        single = hy.hyres(cubes[i].contiguous())
        assert torch.equal(single, outs[i])
        if i == 0:
            ref = O.hyres(s.noisy)
            _compare(s, ref, outs[i].cpu().numpy(), infos[i])


def test_host_api_equals_device_api(hy):
    s = synth.make_cube("small", 0)
    d = hy.hyres(dev(s.noisy)).cpu().numpy()
    h, info = hy.hyres_host(s.noisy, return_info=True)
    assert np.array_equal(d, h)
    pinned = torch.from_numpy(s.noisy).pin_memory()
    h2 = hy.hyres_host(pinned)
    assert np.array_equal(d, h2.numpy())


def test_host_stream_equals_device_api(hy):
    """Streaming host path (overlapped H2D / compute / D2H, two device slots):
    every output equals the device-API result of its own cube, including when
    consecutive cubes differ and n exceeds the two slots."""
    cubes = [synth.make_cube("tiny", seed).noisy for seed in range(5)]
    ref = [hy.hyres(dev(c)).cpu().numpy() for c in cubes]
    pins = [torch.from_numpy(c).pin_memory() for c in cubes]
    outs, infos = hy.hyres_host_stream(pins, return_info=True)
    for r, o, info in zip(ref, outs, infos):
        assert np.array_equal(r, o.numpy())
        assert info["rank"] >= 1
    assert hy.hyres_host_stream([]) == []


def test_deterministic_and_in_place(hy):
    s = synth.make_cube("tiny", 0)
    a = hy.hyres(dev(s.noisy))
    b = hy.hyres(dev(s.noisy))
    assert torch.equal(a, b)
    x = dev(s.noisy)
    hy.hyres(x, out=x)
    assert torch.equal(x, a)


@pytest.mark.parametrize("taps,levels,keep_ll", [(2, 0, False), (8, 0, False), (16, 1, False), (16, 0, True)])
def test_params_variants_match_oracle(hy, taps, levels, keep_ll):
    s = synth.make_cube("tiny", 0)
    ref = O.hyres(s.noisy, taps=taps, levels=levels, keep_ll=keep_ll)
    out, info = hy.hyres(dev(s.noisy), taps=taps, levels=levels, keep_ll=keep_ll, return_info=True)
    _compare(s, ref, out.cpu().numpy(), info)


def test_chunk_boundary_rank(hy):
    """Small chunks force several projection chunks (rank walk across chunk edges)."""
    s = synth.make_cube("small", 0)
    ref = O.hyres(s.noisy)
    for chunk in (1, 2, 3):
        out, info = hy.hyres(dev(s.noisy), chunk=chunk, return_info=True)
        assert info["chunks_run"] >= (ref.rank + 1 + chunk - 1) // chunk
        _compare(s, ref, out.cpu().numpy(), info)


def test_noiseless_low_rank(hy):
    s = synth.low_rank_cube(64, 64, 32, rank=4, seed=11)
    ref = O.hyres(s.clean)
    out, info = hy.hyres(dev(s.clean), return_info=True)
    assert info["rank"] == 4 == ref.rank
    assert metrics.rel_l2(s.clean, out.cpu().numpy()) < 1e-4


def test_odd_ragged_shapes(hy):
    for (b, r, c, seed) in [(3, 17, 33, 0), (9, 31, 29, 1), (40, 65, 127, 2), (256, 40, 40, 3)]:
        s = synth.low_rank_cube(r, c, b, rank=min(3, b - 1), seed=seed, snr_db=20.0)
        ref = O.hyres(s.noisy)
        out, info = hy.hyres(dev(s.noisy), return_info=True)
        assert info["rank"] == ref.rank, (b, r, c)
        assert metrics.rel_l2(ref.out, out.cpu().numpy()) <= REL_L2, (b, r, c)


def test_invariances_on_gpu(hy):
    s = synth.make_cube("tiny", 0)
    base = hy.hyres(dev(s.noisy)).cpu().numpy()
    perm = np.random.default_rng(8).permutation(s.noisy.shape[0])
    assert metrics.rel_l2(base[perm], hy.hyres(dev(s.noisy[perm])).cpu().numpy()) < 1e-5
    tr = np.ascontiguousarray(s.noisy.transpose(0, 2, 1))
    assert metrics.rel_l2(base.transpose(0, 2, 1), hy.hyres(dev(tr)).cpu().numpy()) < 1e-5
    sh = np.roll(s.noisy, (12, -8), axis=(1, 2))
    assert metrics.rel_l2(np.roll(base, (12, -8), axis=(1, 2)), hy.hyres(dev(sh)).cpu().numpy()) < 1e-5
    sh1 = np.roll(s.noisy, 1, axis=2)
    assert metrics.rel_l2(np.roll(base, 1, axis=2), hy.hyres(dev(sh1)).cpu().numpy()) > 1e-4


def test_zero_cube_and_errors(hy):
    z = torch.zeros((8, 16, 16), device="cuda")
    out = hy.hyres(z)
    assert torch.count_nonzero(out) == 0
    bad = torch.ones((8, 16, 16), device="cuda")
    bad[2, 3, 4] = float("nan")
    with pytest.raises(hy.HydeError) as ei:
        hy.hyres(bad)
    assert ei.value.status == 3
    with pytest.raises(hy.HydeError) as ei:
        hy.hyres(torch.ones((2, 16, 16), device="cuda"))
    assert ei.value.status == 2
    with pytest.raises(hy.HydeError):
        hy.hyres(torch.ones((8, 4, 2), device="cuda"))      # pixels <= bands
    with pytest.raises(hy.HydeError):
        hy.hyres(torch.ones((8, 16, 16), device="cuda"), taps=6)
    with pytest.raises(hy.HydeError):
        hy.hyres(torch.ones((8, 16, 16), device="cuda"), levels=7)
    with pytest.raises(hy.HydeError):
        hy.hyres(torch.ones((8, 16, 16)))                   # CPU tensor: no CPU path


def test_hyres_max_bands_simt_gram_path(hy):
    """B = 256 (the largest supported; above the tensor-core Gram's 224-band tiling, so
    K1 falls back to the fp64 SIMT Gram) end to end against the oracle."""
    s = synth.low_rank_cube(40, 36, 256, rank=3, seed=5, snr_db=20.0)
    ref = O.hyres(s.noisy)
    out, info = hy.hyres(torch.from_numpy(s.noisy).cuda(), return_info=True)
    assert info["rank"] == ref.rank
    assert metrics.rel_l2(ref.out, out.cpu().numpy()) <= 1e-4


def _hot(cube, mult, seed):
    """One pixel at mult x the band RMS in every band (a hot / specular pixel)."""
    cube = cube.copy()
    b, r, c = cube.shape
    rms = np.sqrt(np.mean(cube.reshape(b, -1).astype(np.float64) ** 2, axis=1))
    i, j = np.random.default_rng(100 + seed).integers(0, min(r, c), 2)
    cube[:, i, j] = (mult * rms).astype(np.float32)
    return cube


@pytest.mark.parametrize("seed", [0, 1, 2])
@pytest.mark.parametrize("mult", [10.0, 30.0, 100.0, 1000.0])
def test_hyres_outlier_bands_match_oracle(hy, seed, mult):
    """VERDICT r01 item 1 / PAPER.md:261-263: a hot pixel at 10-1000 x the band RMS in
    every band must not cost parity (north_star: rel L2 <= 1e-4, 0.01 dB, equal r*)."""
    s = synth.make_cube("tiny", seed)
    cube = _hot(s.noisy, mult, seed)
    ref = O.hyres(cube)
    out, info = hy.hyres(dev(cube), return_info=True)
    _compare(synth.Sample(s.cfg, s.seed, s.clean, cube), ref, out.cpu().numpy(), info)
    sig = hy.estimate_noise(dev(cube))
    assert np.max(np.abs(sig.cpu().numpy() / ref.sigma - 1)) < 1e-5


def test_hyres_spike_band_small_matches_oracle(hy):
    """small cube: one band with a single 1e3 x spike, plus a 3000 x hot pixel and a dead band."""
    s = synth.make_cube("small", 0)
    cube = _hot(s.noisy, 3000.0, 7)
    b = cube.shape[0]
    rms = np.sqrt(np.mean(cube.reshape(b, -1).astype(np.float64) ** 2, axis=1))
    cube[50, 70, 70] = np.float32(1e3 * rms[50])
    ref = O.hyres(cube)
    out, info = hy.hyres(dev(cube), return_info=True)
    _compare(synth.Sample(s.cfg, s.seed, s.clean, cube), ref, out.cpu().numpy(), info)


@pytest.mark.slow
def test_hyres_large_hot_pixel_matches_oracle(hy):
    s = synth.make_cube("large", 0)
    cube = _hot(s.noisy, 100.0, 3)
    ref = O.hyres(cube)
    out, info = hy.hyres(dev(cube), return_info=True)
    _compare(synth.Sample(s.cfg, s.seed, s.clean, cube), ref, out.cpu().numpy(), info)


def test_rank_walk_to_last_component(hy):
    """The rank walk reaches k = B (r* = B - 1, the largest r* the rule can give: the
    smallest eigenvalue of G_w is <= 1, so E_post,B <= N <= N_c -- pinned in
    test_oracle_pins.py::test_last_component_always_fails), across chunk edges."""
    s = synth.low_rank_cube(64, 64, 4, rank=4, seed=3)
    ref = O.hyres(s.clean)
    assert ref.rank == 3 and len(ref.e_post) == 4
    for chunk in (1, 2, 16):
        out, info = hy.hyres(dev(s.clean), chunk=chunk, return_info=True)
        assert info["rank"] == 3 and info["comps"] == 4
        assert metrics.rel_l2(ref.out, out.cpu().numpy()) <= REL_L2


def test_validate_flag_fails_fast_on_nonfinite(hy):
    """flags bit1 HYDE_VALIDATE: a synchronous finiteness pass before any work;
    finite input gives the same result as without the flag."""
    s = synth.make_cube("tiny", 0)
    x = dev(s.noisy)
    assert torch.equal(hy.hyres(x, validate=True), hy.hyres(x))
    bad = x.clone()
    bad[5, 9, 9] = float("inf")
    for fn in (lambda t: hy.hyres(t, validate=True),
               lambda t: hy.hyres_batched(torch.stack([x, t]), validate=True)):
        with pytest.raises(hy.HydeError) as ei:
            fn(bad)
        assert ei.value.status == 3


def test_batched_phased_needs_second_chunk(hy):
    """Phased batched path: a cube whose rank rule needs more than the first chunk of 4
    components (a noiseless rank-6 cube, r* = 6) is finished by the chunked walk; every
    output equals the single-cube result bit for bit."""
    cubes = [synth.make_cube("tiny", 0).noisy, synth.low_rank_cube(64, 64, 32, rank=6, seed=2).clean,
             synth.make_cube("tiny", 3).noisy]
    x = dev(np.stack(cubes))
    outs, infos = hy.hyres_batched(x, return_info=True)
    for i in range(len(cubes)):
        single, info = hy.hyres(x[i].contiguous(), return_info=True)
        assert torch.equal(single, outs[i]), i
        assert infos[i]["rank"] == info["rank"]
    assert max(i["rank"] for i in infos) >= 4


def _lanczos(hy, enable, max_steps=0):
    assert hy._lib.lib().hyde_debug_eig_lanczos(enable, max_steps) == 0


@pytest.mark.parametrize("name", ["tiny", "small", "medium", "wide"])
def test_first_chunk_lanczos_householder_and_fallback(hy, name):
    """K2's first chunk three ways: Lanczos (phase 2L, the default), the Householder
    path (phase 2 + 3), and Lanczos capped at 5 steps -- below convergence, so the
    kernel falls back to Householder in place.  Same rank, outputs within 1e-6 of
    each other, each within the oracle tolerance (wide: r* > the first chunk, so the
    tridiagonal rerun after Lanczos serves the second chunk)."""
    s = synth.make_cube(name, 0)
    ref = O.hyres(s.noisy)
    x = dev(s.noisy)
    outs = []
    try:
        for en, cap in ((1, 0), (0, 0), (1, 5)):
            _lanczos(hy, en, cap)
            out, info = hy.hyres(x, return_info=True)
            o = out.cpu().numpy()
            _compare(s, ref, o, info)
            outs.append(o)
    finally:
        _lanczos(hy, 1, 0)
    assert metrics.rel_l2(outs[1], outs[0]) <= 1e-6
    assert metrics.rel_l2(outs[1], outs[2]) <= 1e-6
