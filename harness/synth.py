"""Seeded synthetic hyperspectral cubes shaped like the paper's workloads.

This module is the ONLY code shared by the oracle (``oracle/``) and the CUDA
path's tests/bench: it draws inputs and holds none of HyRes' arithmetic.

The paper's experiments use the Houston 2013 cube with additive Gaussian noise
(Sec. 3 "Experiments"); that cube is not available here, so
the five ``BASELINE.json`` configs stand in for it (``wide`` has the Houston
shape).  The recipe follows SURVEY.md §8(d) and is restated in DESIGN.md §3:

1. K endmember spectra, each a sum of 3 Gaussian bumps (centre ~ U(0, B),
   width ~ U(B/16, B/4), amplitude ~ U(0.2, 1)), divided by its max.
2. Abundances: per-pixel Dirichlet(1_K), then a 5x5 box filter (tiny), a
   Gaussian sigma = 3 px filter (small/medium/large/batched), or for ``wide``
   a 200-seed Voronoi partition with one Dirichlet vector per region, then the
   Gaussian blur.  Filters are linear and sum-preserving, so the abundances
   still sum to one.
3. Clean cube X = sum_k s_k (x) A_k, stored band-sequential (BSQ) float32
   ``[bands][rows][cols]`` (SPEC.md:22-27 HsiCube, BSQ order SPEC.md:23).
4. Noise (PAPER.md:84 lists the simulators; SPEC.md:208-252 defines them):
   i.i.d. Gaussian at a target SNR (sigma = sqrt(mean(X^2) / 10^(SNR/10)),
   SPEC.md:211); non-i.i.d. Gaussian with per-band SNR in [lo, hi];
   salt-and-pepper and dead columns for ``medium``.

All randomness comes from ``numpy.random.default_rng(seed)`` (PCG64), drawn in
the fixed order below, so a (config, seed) pair always yields the same bytes.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional

import numpy as np
from scipy import ndimage


@dataclass(frozen=True)
class CubeConfig:
    name: str
    rows: int
    cols: int
    bands: int
    endmembers: int
    abundance: str                  # "box5" | "gauss3" | "voronoi_gauss3"
    noise: str                      # "iid" | "noniid"
    snr_db: float = 20.0            # iid target SNR
    snr_lo_db: float = 10.0         # noniid band-SNR range
    snr_hi_db: float = 30.0
    sparse: bool = False            # medium: salt&pepper + dead columns in 10 % of bands
    voronoi_seeds: int = 200
    batch: int = 1                  # number of independent cubes (seeds seed0 .. seed0+batch-1)
    description: str = ""

    @property
    def pixels(self) -> int:
        return self.rows * self.cols

    @property
    def voxels(self) -> int:
        return self.rows * self.cols * self.bands


# BASELINE.json "configs" (five strings; the fifth names two workloads).
CONFIGS = {
    "tiny": CubeConfig("tiny", 64, 64, 32, 4, "box5", "iid", snr_db=20.0,
                       description="BASELINE.json configs[0]"),
    "small": CubeConfig("small", 145, 145, 200, 8, "gauss3", "noniid", snr_lo_db=10.0, snr_hi_db=30.0,
                        description="BASELINE.json configs[1]"),
    "medium": CubeConfig("medium", 610, 340, 103, 9, "gauss3", "iid", snr_db=10.0, sparse=True,
                         description="BASELINE.json configs[2]"),
    "wide": CubeConfig("wide", 349, 1905, 144, 12, "voronoi_gauss3", "iid", snr_db=10.0,
                       description="BASELINE.json configs[3] (Houston 2013 shape)"),
    "large": CubeConfig("large", 1024, 1024, 224, 16, "gauss3", "noniid", snr_lo_db=5.0, snr_hi_db=25.0,
                        description="BASELINE.json configs[4], first workload (north_star target)"),
    "batched": CubeConfig("batched", 256, 256, 191, 16, "gauss3", "noniid", snr_lo_db=5.0, snr_hi_db=25.0,
                          batch=64, description="BASELINE.json configs[4], second workload (64 cubes, seeds 0-63)"),
}


def endmember_spectra(rng: np.random.Generator, k: int, bands: int) -> np.ndarray:
    """K smooth spectra in (0, 1], shape (K, B): sums of 3 Gaussian bumps."""
    b = np.arange(bands, dtype=np.float64)
    centres = rng.uniform(0.0, bands, size=(k, 3))
    widths = rng.uniform(bands / 16.0, bands / 4.0, size=(k, 3))
    amps = rng.uniform(0.2, 1.0, size=(k, 3))
    s = np.zeros((k, bands))
    for j in range(3):
        s += amps[:, j:j + 1] * np.exp(-0.5 * ((b[None, :] - centres[:, j:j + 1]) / widths[:, j:j + 1]) ** 2)
    s /= s.max(axis=1, keepdims=True)
    return s


def abundances(rng: np.random.Generator, cfg: CubeConfig) -> np.ndarray:
    """Abundance maps, shape (K, R, C), non-negative, summing to one per pixel."""
    k, r, c = cfg.endmembers, cfg.rows, cfg.cols
    if cfg.abundance == "voronoi_gauss3":
        seeds_rc = rng.uniform(0.0, 1.0, size=(cfg.voronoi_seeds, 2)) * np.array([r, c])
        region_ab = rng.dirichlet(np.ones(k), size=cfg.voronoi_seeds)          # (S, K)
        # nearest seed at pixel centres, computed row by row to bound memory
        labels = np.empty((r, c), dtype=np.int64)
        cc = np.arange(c) + 0.5
        for i in range(r):
            d2 = (i + 0.5 - seeds_rc[:, 0:1]) ** 2 + (cc[None, :] - seeds_rc[:, 1:2]) ** 2  # (S, C)
            labels[i] = np.argmin(d2, axis=0)
        a = region_ab[labels].transpose(2, 0, 1)                                  # (K, R, C)
    else:
        a = rng.dirichlet(np.ones(k), size=(r, c)).transpose(2, 0, 1)          # (K, R, C)
    a = np.ascontiguousarray(a)
    out = np.empty_like(a)
    for j in range(k):
        if cfg.abundance == "box5":
            out[j] = ndimage.uniform_filter(a[j], size=5, mode="reflect")
        else:
            out[j] = ndimage.gaussian_filter(a[j], sigma=3.0, mode="reflect")
    return out


def clean_cube(rng: np.random.Generator, cfg: CubeConfig) -> np.ndarray:
    """Noise-free BSQ cube, float32 (B, R, C)."""
    s = endmember_spectra(rng, cfg.endmembers, cfg.bands)                     # (K, B)
    a = abundances(rng, cfg)                                                    # (K, R, C)
    x = (s.T.astype(np.float32) @ a.reshape(cfg.endmembers, -1).astype(np.float32))
    return x.reshape(cfg.bands, cfg.rows, cfg.cols)


def add_noise(rng: np.random.Generator, x: np.ndarray, cfg: CubeConfig) -> np.ndarray:
    """Additive noise per cfg; returns a new float32 BSQ cube."""
    b = x.shape[0]
    flat = x.reshape(b, -1)
    if cfg.noise == "iid":
        p = float(np.mean(flat.astype(np.float64) ** 2))
        sig = np.full(b, np.sqrt(p / 10.0 ** (cfg.snr_db / 10.0)))
    elif cfg.noise == "noniid":
        pb = np.mean(flat.astype(np.float64) ** 2, axis=1)
        u = rng.uniform(0.0, 1.0, size=b)
        sig = u * np.sqrt(pb / 10.0 ** (cfg.snr_lo_db / 10.0)) + (1.0 - u) * np.sqrt(pb / 10.0 ** (cfg.snr_hi_db / 10.0))
    else:
        raise ValueError(cfg.noise)
    y = np.empty_like(x)
    yf = y.reshape(b, -1)
    for i in range(b):  # band by band to bound peak memory at `large`
        yf[i] = flat[i] + (sig[i] * rng.standard_normal(flat.shape[1])).astype(np.float32)
    if cfg.sparse:
        nb = int(round(0.1 * b))
        bands = rng.choice(b, size=nb, replace=False)
        for bi in bands:
            img = y[bi]
            lo, hi = img.min(), img.max()
            u = rng.uniform(0.0, 1.0, size=img.shape)
            img[u < 0.025] = lo
            img[(u >= 0.025) & (u < 0.05)] = hi
            dead = rng.choice(img.shape[1], size=10, replace=False)
            img[:, dead] = 0.0
    return y


@dataclass
class Sample:
    cfg: CubeConfig
    seed: int
    clean: np.ndarray   # float32 (B, R, C)
    noisy: np.ndarray   # float32 (B, R, C)


def make_cube(cfg: CubeConfig | str, seed: int = 0) -> Sample:
    """Generate one (clean, noisy) pair; same (cfg, seed) -> identical bytes."""
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    rng = np.random.default_rng(seed)
    x = clean_cube(rng, cfg)
    y = add_noise(rng, x, cfg)
    return Sample(cfg, seed, x, y)


def make_batch(cfg: CubeConfig | str, seeds) -> np.ndarray:
    """Noisy cubes for a list of seeds, stacked (batch, B, R, C) float32."""
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    return np.stack([make_cube(cfg, s).noisy for s in seeds])


def low_rank_cube(rows: int, cols: int, bands: int, rank: int, seed: int = 0,
                  snr_db: Optional[float] = None) -> Sample:
    """Rank-`rank` cube from random non-negative factors (SPEC.md:545 `synth --kind lowrank`);
    optional i.i.d. Gaussian noise at `snr_db`."""
    rng = np.random.default_rng(seed)
    s = endmember_spectra(rng, rank, bands)
    a = rng.dirichlet(np.ones(rank), size=(rows, cols)).transpose(2, 0, 1)
    for j in range(rank):
        a[j] = ndimage.gaussian_filter(a[j], sigma=2.0, mode="wrap")
    x = (s.T @ a.reshape(rank, -1)).astype(np.float32).reshape(bands, rows, cols)
    if snr_db is None:
        y = x.copy()
    else:
        sig = np.sqrt(float(np.mean(x.astype(np.float64) ** 2)) / 10.0 ** (snr_db / 10.0))
        y = (x + sig * rng.standard_normal(x.shape)).astype(np.float32)
    cfg = CubeConfig(f"lowrank{rank}", rows, cols, bands, rank, "gauss2", "iid" if snr_db else "none")
    return Sample(cfg, seed, x, y)
