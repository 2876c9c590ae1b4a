"""Stage entry points (hyde_k_*) for stage-isolated parity tests.

Each consumes / produces the oracle's intermediate layout (oracle/hyres_ref.py):
  gram       Y (B, N) fp32            -> G (B, B) fp64
  eig        G, N                     -> sigma (B,), lam (B,) descending, V (B, ncomp)
  project    Y, W (B, ncomp) fp32     -> E (ncomp, N)
  dwt_fwd    images (count, R, C)     -> coeffs (count, N_c): level 1..L x (LH, HL, HH), LL_L
  sure       coeffs (in place)        -> kstar, tstar (count, 3L+1), e_post (count,)
  idwt       coeffs                   -> images
  wavelet_shrink images (count, R, C)  -> denoised images, kstar, tstar, e_post (A4 -> A5 -> A6a)
  reconstruct E (r, N), U (B, r)      -> out (B, N)
"""
from __future__ import annotations

import ctypes

from ._lib import check, lib
from . import _cube, _stream, _torch, handle


def _h(t):
    return handle(t.device.index)


def auto_levels(rows, cols, taps=16) -> int:
    return int(lib().hyde_auto_levels(rows, cols, taps))


def coeff_count(rows, cols, levels) -> int:
    return int(lib().hyde_dwt_coeff_count(rows, cols, levels))


def filter_lowpass(taps=16):
    import numpy as np
    buf = (ctypes.c_double * taps)()
    check(lib().hyde_filter(taps, buf))
    return np.array(buf[:], dtype=np.float64)


def gram(cube):
    torch = _torch()
    b = cube.shape[0]
    n = cube[0].numel()
    y = cube.contiguous()
    g = torch.empty((b, b), dtype=torch.float64, device=cube.device)
    h = _h(cube)
    check(lib().hyde_k_gram(h, y.data_ptr(), n, b, g.data_ptr(), _stream(cube)), h)
    return g


def gram_quant(cube):
    """Quantisation of the last `gram(cube)` call on this device: per band the fp32
    1/step inv_s and the integer centre c (q = rint(y inv_s) - c), and the number of
    pixels added exactly (flagged); flagged = -1 when the fp64 SIMT path ran."""
    import numpy as np
    b = cube.shape[0]
    n = cube[0].numel()
    inv_s = (ctypes.c_float * b)()
    cen = (ctypes.c_int * b)()
    nf = ctypes.c_longlong(0)
    h = _h(cube)
    check(lib().hyde_debug_gram_quant(h, n, b, inv_s, cen, ctypes.byref(nf)), h)
    return np.array(inv_s[:], dtype=np.float32), np.array(cen[:], dtype=np.int64), int(nf.value)


def eig(g, n_pixels, ncomp, ridge=1e-6, all_lam=True):
    torch = _torch()
    b = g.shape[0]
    g = g.contiguous()
    sigma = torch.empty(b, dtype=torch.float64, device=g.device)
    lam = torch.empty(b, dtype=torch.float64, device=g.device) if all_lam else None
    V = torch.empty((b, max(ncomp, 1)), dtype=torch.float64, device=g.device)
    h = _h(g)
    check(lib().hyde_k_eig(h, g.data_ptr(), int(n_pixels), b, float(ridge), int(ncomp), sigma.data_ptr(),
                           lam.data_ptr() if lam is not None else None, V.data_ptr(), _stream(g)), h)
    return sigma, lam, V[:, :ncomp]


def project(cube, W):
    torch = _torch()
    b = cube.shape[0]
    n = cube[0].numel()
    W = W.contiguous().to(torch.float32)
    k = W.shape[1]
    E = torch.empty((k, n), dtype=torch.float32, device=cube.device)
    h = _h(cube)
    check(lib().hyde_k_project(h, cube.data_ptr(), n, b, W.data_ptr(), k, E.data_ptr(), _stream(cube)), h)
    return E


def dwt_fwd(images, levels, taps=16):
    torch = _torch()
    _cube(images, "images")
    cnt, r, c = images.shape
    nc = coeff_count(r, c, levels)
    co = torch.empty((cnt, nc), dtype=torch.float32, device=images.device)
    h = _h(images)
    check(lib().hyde_k_dwt_fwd(h, images.data_ptr(), cnt, r, c, levels, taps, co.data_ptr(), _stream(images)), h)
    return co


def sure(coeffs, rows, cols, levels, keep_ll=False):
    """In-place soft threshold of coeffs (count, N_c); returns kstar, tstar, e_post."""
    torch = _torch()
    cnt = coeffs.shape[0]
    nsub = 3 * levels + 1
    ks = torch.empty((cnt, nsub), dtype=torch.int32, device=coeffs.device)
    ts = torch.empty((cnt, nsub), dtype=torch.float32, device=coeffs.device)
    ep = torch.empty(cnt, dtype=torch.float64, device=coeffs.device)
    h = _h(coeffs)
    check(lib().hyde_k_sure(h, coeffs.data_ptr(), cnt, rows, cols, levels, 1 if keep_ll else 0, ks.data_ptr(),
                            ts.data_ptr(), ep.data_ptr(), _stream(coeffs)), h)
    return ks, ts, ep


def idwt(coeffs, rows, cols, levels, taps=16):
    torch = _torch()
    cnt = coeffs.shape[0]
    out = torch.empty((cnt, rows, cols), dtype=torch.float32, device=coeffs.device)
    h = _h(coeffs)
    check(lib().hyde_k_idwt(h, coeffs.contiguous().data_ptr(), cnt, rows, cols, levels, taps, out.data_ptr(),
                            _stream(coeffs)), h)
    return out


def wavelet_shrink(images, levels, taps=16, keep_ll=False, out=None, stats=True, analyze_only=False):
    """A4 -> A5 -> A6a on a batch of images, as the hot path runs them (hyde_wavelet_shrink).
    Returns out (count, R, C) and, with stats, kstar / tstar (count, 3L+1) and e_post (count,).
    analyze_only: DWT + SURE only (no IDWT; out is None)."""
    torch = _torch()
    _cube(images, "images")
    cnt, r, c = images.shape
    nsub = 3 * levels + 1
    if out is None and not analyze_only:
        out = torch.empty_like(images)
    ks = torch.empty((cnt, nsub), dtype=torch.int32, device=images.device) if stats else None
    ts = torch.empty((cnt, nsub), dtype=torch.float32, device=images.device) if stats else None
    ep = torch.empty(cnt, dtype=torch.float64, device=images.device) if stats else None
    h = _h(images)
    p = lambda t: t.data_ptr() if t is not None else None
    check(lib().hyde_wavelet_shrink(h, images.data_ptr(), cnt, r, c, levels, taps, 1 if keep_ll else 0,
                                    None if analyze_only else out.data_ptr(), p(ks), p(ts), p(ep), _stream(images)), h)
    return (out, ks, ts, ep) if stats else out


def reconstruct(E, U, bands_shape=None):
    torch = _torch()
    r, n = E.shape
    b = U.shape[0]
    U = U.contiguous().to(torch.float32)
    out = torch.empty((b, n), dtype=torch.float32, device=E.device)
    h = _h(E)
    check(lib().hyde_k_reconstruct(h, E.contiguous().data_ptr(), n, b, U.data_ptr(), U.shape[1], r,
                                   out.data_ptr(), _stream(E)), h)
    return out if bands_shape is None else out.reshape(bands_shape)
