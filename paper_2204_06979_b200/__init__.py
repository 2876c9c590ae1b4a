"""B200-native HyRes (HyDe, arXiv 2204.06979): Python binding of libhyde.so.

PyTorch supplies device memory and the current CUDA stream; every stage of the
method runs in libhyde's sm_100a kernels behind the C-ABI of include/hyde.h.
Inputs must be CUDA float32 tensors in BSQ layout (bands, rows, cols); there
is no CPU path.
"""
from __future__ import annotations

import ctypes
from typing import Dict, Optional, Tuple

from . import _lib
from ._lib import HydeError, Info, Params, check, lib, make_params

__all__ = ["hyres", "hyres_batched", "hyres_host", "hyres_host_stream", "hyres_sharded", "NcclComm",
           "nccl_comm_single", "make_comm", "slab_rows", "component_owner", "estimate_noise", "workspace_size",
           "HydeError", "stages", "version"]

_handles: Dict[int, int] = {}


def version() -> str:
    return lib().hyde_version().decode()


def _torch():
    import torch
    return torch


def handle(device: int) -> int:
    h = _handles.get(device)
    if h is None:
        hv = ctypes.c_void_p()
        check(lib().hyde_create(ctypes.byref(hv), int(device)))
        h = hv.value
        _handles[device] = h
    return h


def _stream(t) -> int:
    torch = _torch()
    return torch.cuda.current_stream(t.device).cuda_stream


def _cube(t, name="cube", ndim=3):
    torch = _torch()
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise HydeError(2, f"{name} must be a CUDA tensor (no CPU path)")
    if t.dtype != torch.float32:
        raise HydeError(2, f"{name} must be float32")
    if t.dim() != ndim:
        raise HydeError(2, f"{name} must have {ndim} dims")
    if not t.is_contiguous():
        raise HydeError(2, f"{name} must be contiguous")
    return t


def hyres(cube, out=None, *, taps=16, levels=0, chunk=16, ridge=1e-6, keep_ll=False,
          return_info=False, validate=False):
    """HyRes denoising of one BSQ cube (bands, rows, cols) -> same shape.
    validate=True: HYDE_VALIDATE (fail fast on non-finite input, one extra read)."""
    torch = _torch()
    _cube(cube)
    b, r, c = cube.shape
    if out is None:
        out = torch.empty_like(cube)
    else:
        _cube(out, "out")
    p = make_params(taps, levels, chunk, ridge, keep_ll, validate)
    info = Info()
    h = handle(cube.device.index)
    check(lib().hyde_hyres_ex(h, cube.data_ptr(), r, c, b, out.data_ptr(), ctypes.byref(p),
                              ctypes.byref(info), _stream(cube)), h)
    return (out, info.as_dict()) if return_info else out


def hyres_batched(cubes, out=None, *, taps=16, levels=0, chunk=16, ridge=1e-6, keep_ll=False,
                  return_info=False, validate=False):
    """`batch` independent cubes (batch, bands, rows, cols)."""
    torch = _torch()
    _cube(cubes, "cubes", 4)
    n, b, r, c = cubes.shape
    if out is None:
        out = torch.empty_like(cubes)
    p = make_params(taps, levels, chunk, ridge, keep_ll, validate)
    infos = (Info * max(n, 1))()
    h = handle(cubes.device.index)
    check(lib().hyde_hyres_batched(h, cubes.data_ptr(), n, r, c, b, out.data_ptr(), ctypes.byref(p),
                                   infos, _stream(cubes)), h)
    return (out, [infos[i].as_dict() for i in range(n)]) if return_info else out


def hyres_host(cube_np, out_np=None, *, device=0, taps=16, levels=0, chunk=16, ridge=1e-6,
               keep_ll=False, return_info=False):
    """End-to-end call with HOST buffers (numpy float32, C-contiguous; pinned or pageable):
    the library copies the cube in, denoises, copies the result out."""
    import numpy as np
    torch = _torch()
    a = cube_np
    if isinstance(a, torch.Tensor):
        if a.is_cuda or a.dtype != torch.float32 or not a.is_contiguous():
            raise HydeError(2, "host cube must be a contiguous float32 CPU tensor")
        b, r, c = a.shape
        out = torch.empty_like(a) if out_np is None else out_np
        src, dst = a.data_ptr(), out.data_ptr()
    else:
        a = np.ascontiguousarray(a, dtype=np.float32)
        b, r, c = a.shape
        out = np.empty_like(a) if out_np is None else out_np
        src, dst = a.ctypes.data, out.ctypes.data
    p = make_params(taps, levels, chunk, ridge, keep_ll)
    info = Info()
    h = handle(device)
    stream = torch.cuda.current_stream(device).cuda_stream
    check(lib().hyde_hyres_host(h, src, r, c, b, dst, ctypes.byref(p), ctypes.byref(info), stream), h)
    return (out, info.as_dict()) if return_info else out


def hyres_host_stream(cubes, outs=None, *, device=0, taps=16, levels=0, chunk=16, ridge=1e-6, keep_ll=False,
                      return_info=False):
    """Streaming end-to-end path over a list of HOST cubes (contiguous float32
    CPU tensors, ideally pinned): the H2D copy of cube i+1 and the D2H copy of
    cube i-1 overlap the denoising of cube i (include/hyde.h
    hyde_hyres_host_stream).  Returns the list of output host tensors."""
    torch = _torch()
    n = len(cubes)
    if n == 0:
        return ([], []) if return_info else []
    if outs is None:
        outs = [torch.empty_like(c) for c in cubes]
    for c in list(cubes) + list(outs):
        if not isinstance(c, torch.Tensor) or c.is_cuda or c.dtype != torch.float32 or not c.is_contiguous():
            raise HydeError(2, "host cubes must be contiguous float32 CPU tensors")
    b, r, c = cubes[0].shape
    src = (ctypes.c_void_p * max(n, 1))(*[x.data_ptr() for x in cubes])
    dst = (ctypes.c_void_p * max(n, 1))(*[x.data_ptr() for x in outs])
    p = make_params(taps, levels, chunk, ridge, keep_ll)
    infos = (Info * max(n, 1))()
    h = handle(device)
    stream = torch.cuda.current_stream(device).cuda_stream
    check(lib().hyde_hyres_host_stream(h, src, dst, n, r, c, b, ctypes.byref(p), infos, stream), h)
    return (outs, [infos[i].as_dict() for i in range(n)]) if return_info else outs


class _DevBuf:
    """Zero-copy view of a raw device buffer for torch.as_tensor (CUDA array interface)."""

    def __init__(self, ptr, count, typestr):
        self.__cuda_array_interface__ = {"shape": (int(count),), "typestr": typestr, "data": (int(ptr), False),
                                         "version": 3, "strides": None}


def dev_view(ptr, count, typestr):
    return _torch().as_tensor(_DevBuf(ptr, count, typestr), device="cuda")


def slab_rows(rows, rank, world):
    """Pixel rows [r0, r1) of rank `rank` in the sharded path (hyde_shard_rows)."""
    r0, nr = ctypes.c_int(0), ctypes.c_int(0)
    if lib().hyde_shard_rows(int(rows), int(world), int(rank), ctypes.byref(r0), ctypes.byref(nr)) != 0:
        raise HydeError(2, "bad rank / world")
    return r0.value, r0.value + nr.value


def component_owner(k, world):
    """Rank that owns candidate component k (0-based) in the sharded wavelet stage (hyde_shard_owner)."""
    return int(lib().hyde_shard_owner(int(k), int(world)))


def make_comm(rank, world, allreduce_sum_f64, sendrecv):
    """Wrap two Python collectives into a hyde_comm (hyde_hyres_sharded_cb):
    allreduce_sum_f64(t, stream) sums a float64 device view in place over the
    ranks; sendrecv(sends, recvs, stream) gets lists of (peer, uint8 device view)
    -- between two ranks the i-th send matches the i-th receive.  Keep the
    returned object alive for the duration of the call."""
    def asum(user, buf, count, stream):
        try:
            allreduce_sum_f64(dev_view(buf, count, "<f8"), stream)
            return 0
        except Exception:  # noqa: BLE001
            return 1

    def sr(user, ns, sends, nr, recvs, stream):
        try:
            s = [(sends[i].peer, dev_view(sends[i].buf, sends[i].bytes, "|u1")) for i in range(ns)]
            r = [(recvs[i].peer, dev_view(recvs[i].buf, recvs[i].bytes, "|u1")) for i in range(nr)]
            sendrecv(s, r, stream)
            return 0
        except Exception:  # noqa: BLE001
            return 1

    fns = (_lib.ALLREDUCE_FN(asum), _lib.SENDRECV_FN(sr))
    c = _lib.Comm(rank, world, None, *fns)
    c._keep = fns
    return c


class NcclComm:
    """A libhyde NCCL communicator over the ranks of a torch.distributed group:
    rank 0 draws the ncclUniqueId (hyde_nccl_unique_id), the group broadcasts
    it, every rank calls hyde_nccl_comm_init on its current CUDA device.  The
    collectives of hyde_hyres_sharded then run inside libhyde on the call's
    stream (NCCL over NVLink / NVSwitch on a B200 box)."""

    def __init__(self, group=None, device=None):
        import torch.distributed as dist
        torch = _torch()
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.device = torch.cuda.current_device() if device is None else int(device)
        uid = (ctypes.c_ubyte * 128)()
        if self.rank == 0:
            check(lib().hyde_nccl_unique_id(uid))
        t = torch.tensor(list(bytes(uid)), dtype=torch.uint8)
        if dist.get_backend(group) == "nccl":
            t = t.cuda(self.device)
        dist.broadcast(t, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
        raw = bytes(t.cpu().tolist())
        self._uid = (ctypes.c_ubyte * 128).from_buffer_copy(raw)
        c = ctypes.c_void_p()
        check(lib().hyde_nccl_comm_init(ctypes.byref(c), self.world, self.rank, self._uid, self.device))
        self.comm = c.value

    def close(self):
        if self.comm:
            lib().hyde_nccl_comm_destroy(self.comm)
            self.comm = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass


def nccl_comm_single(device=None) -> "NcclComm":
    """World-size-1 NCCL communicator (no process group needed): exercises every
    collective call site of the sharded path on one GPU."""
    torch = _torch()
    obj = NcclComm.__new__(NcclComm)
    obj.rank, obj.world = 0, 1
    obj.device = torch.cuda.current_device() if device is None else int(device)
    uid = (ctypes.c_ubyte * 128)()
    check(lib().hyde_nccl_unique_id(uid))
    obj._uid = uid
    c = ctypes.c_void_p()
    check(lib().hyde_nccl_comm_init(ctypes.byref(c), 1, 0, uid, obj.device))
    obj.comm = c.value
    return obj


def hyres_sharded(local, rows, comm, out=None, *, handle_id=None, taps=16, levels=0, chunk=16, ridge=1e-6,
                  keep_ll=False, return_info=False):
    """Pixel-sharded HyRes of one cube (include/hyde.h hyde_hyres_sharded):
    `local` is this rank's BSQ slab (bands, r1 - r0, cols) with
    (r0, r1) = slab_rows(rows, rank, world); `comm` is an NcclComm (NCCL inside
    libhyde) or a make_comm(...) callback table; returns the denoised slab."""
    torch = _torch()
    _cube(local, "local")
    b, lr, c = local.shape
    if out is None:
        out = torch.empty_like(local)
    r0, r1 = slab_rows(rows, comm.rank, comm.world)
    p = make_params(taps, levels, chunk, ridge, keep_ll)
    info = Info()
    h = handle_id if handle_id is not None else handle(local.device.index)
    if isinstance(comm, NcclComm):
        check(lib().hyde_hyres_sharded(h, comm.comm, local.data_ptr(), lr, r0, rows, c, b, out.data_ptr(),
                                       ctypes.byref(p), ctypes.byref(info), _stream(local)), h)
    else:
        check(lib().hyde_hyres_sharded_cb(h, ctypes.byref(comm), local.data_ptr(), lr, r0, rows, c, b,
                                          out.data_ptr(), ctypes.byref(p), ctypes.byref(info), _stream(local)), h)
    return (out, info.as_dict()) if return_info else out


def estimate_noise(cube, *, return_gram=False, return_residual=False):
    """sigma (bands,) fp64 [, G (bands, bands) fp64] [, residual (bands, rows, cols) fp32]."""
    torch = _torch()
    _cube(cube)
    b, r, c = cube.shape
    sigma = torch.empty(b, dtype=torch.float64, device=cube.device)
    gram = torch.empty((b, b), dtype=torch.float64, device=cube.device) if return_gram else None
    res = torch.empty_like(cube) if return_residual else None
    h = handle(cube.device.index)
    check(lib().hyde_estimate_noise(h, cube.data_ptr(), r, c, b, sigma.data_ptr(),
                                    gram.data_ptr() if gram is not None else None,
                                    res.data_ptr() if res is not None else None, _stream(cube)), h)
    check(lib().hyde_sync_status(h, _stream(cube)), h)
    out = (sigma,)
    if return_gram:
        out += (gram,)
    if return_residual:
        out += (res,)
    return out[0] if len(out) == 1 else out


def l1_spectral(cube, out=None, *, lam=10.0, mu=5.0, max_iters=50, tol=1e-3, return_iters=False):
    """HyMiNoR's second stage (F3; include/hyde.h hyde_l1_spectral)."""
    torch = _torch()
    _cube(cube)
    b, r, c = cube.shape
    if out is None:
        out = torch.empty_like(cube)
    its = torch.empty(r * c, dtype=torch.int32, device=cube.device) if return_iters else None
    h = handle(cube.device.index)
    check(lib().hyde_l1_spectral(h, cube.data_ptr(), r, c, b, out.data_ptr(), float(lam), float(mu), int(max_iters),
                                 float(tol), its.data_ptr() if its is not None else None, _stream(cube)), h)
    return (out, its) if return_iters else out


def hyminor(cube, out=None, *, lam=10.0, mu=5.0, max_iters=50, tol=1e-3, return_info=False):
    """HyMiNoR (F3; include/hyde.h hyde_hyminor): HyRes, then the l1-l1 spectral stage."""
    torch = _torch()
    _cube(cube)
    b, r, c = cube.shape
    if out is None:
        out = torch.empty_like(cube)
    info = Info()
    h = handle(cube.device.index)
    check(lib().hyde_hyminor(h, cube.data_ptr(), r, c, b, out.data_ptr(), float(lam), float(mu), int(max_iters),
                             float(tol), ctypes.byref(info), _stream(cube)), h)
    return (out, info.as_dict()) if return_info else out


def wsrrr(cube, out=None, *, rank=0, lam=-1.0, taps=16, levels=0, max_iters=20, tol=1e-4, components=False):
    """WSRRR (F4; include/hyde.h hyde_wsrrr).  rank 0 = HySime's k, lam < 0 = D17
    default.  Returns dict(out, components (rank, R, C) or None, rank, lam, objective)."""
    torch = _torch()
    _cube(cube)
    b, r, c = cube.shape
    if out is None:
        out = torch.empty_like(cube)
    comps = torch.empty((max(rank, 0) or b, r, c), dtype=torch.float32, device=cube.device) if components else None
    rk, sw = ctypes.c_int(0), ctypes.c_int(0)
    lo = ctypes.c_double(0.0)
    objs = (ctypes.c_double * max(max_iters, 1))()
    h = handle(cube.device.index)
    check(lib().hyde_wsrrr(h, cube.data_ptr(), r, c, b, int(rank), float(lam), int(taps), int(levels), int(max_iters),
                           float(tol), out.data_ptr(), comps.data_ptr() if comps is not None else None,
                           ctypes.byref(rk), ctypes.byref(lo), ctypes.byref(sw), objs, _stream(cube)), h)
    return {"out": out, "components": comps[:rk.value] if comps is not None else None, "rank": int(rk.value),
            "lam": float(lo.value), "objective": [objs[i] for i in range(sw.value)]}


def forpdn(cube, out=None, *, lam=0.0, taps=16, levels=0, return_lambda=False):
    """FORPDN (F2; include/hyde.h hyde_forpdn).  lam = 0: the D16 default from
    {0.1, 1, 10, 100}.  Returns out [, lambda used]."""
    torch = _torch()
    _cube(cube)
    b, r, c = cube.shape
    if out is None:
        out = torch.empty_like(cube)
    lo = ctypes.c_double(0.0)
    h = handle(cube.device.index)
    check(lib().hyde_forpdn(h, cube.data_ptr(), r, c, b, out.data_ptr(), float(lam), int(taps), int(levels),
                            ctypes.byref(lo), _stream(cube)), h)
    return (out, float(lo.value)) if return_lambda else out


def hysime(cube):
    """HySime signal-subspace identification (F1; include/hyde.h hyde_hysime):
    returns dict(k, basis (bands, k) fp64, delta (bands,), mu (bands,), noise_cov (bands, bands))."""
    torch = _torch()
    _cube(cube)
    b, r, c = cube.shape
    dev = cube.device
    basis = torch.zeros((b, b), dtype=torch.float64, device=dev)
    delta = torch.empty(b, dtype=torch.float64, device=dev)
    mu = torch.empty(b, dtype=torch.float64, device=dev)
    ncov = torch.empty((b, b), dtype=torch.float64, device=dev)
    k = ctypes.c_int(0)
    h = handle(dev.index)
    check(lib().hyde_hysime(h, cube.data_ptr(), r, c, b, ctypes.byref(k), basis.data_ptr(), delta.data_ptr(),
                            mu.data_ptr(), ncov.data_ptr(), _stream(cube)), h)
    return {"k": int(k.value), "basis": basis[:, :k.value], "delta": delta, "mu": mu, "noise_cov": ncov}


def workspace_size(rows, cols, bands, batch=1, chunk=16, taps=16, levels=0) -> int:
    p = make_params(taps, levels, chunk)
    return int(lib().hyde_hyres_workspace_size(rows, cols, bands, batch, ctypes.byref(p)))


from . import stages  # noqa: E402


def profile_enable(device: int = 0, on: bool = True) -> None:
    """Record per-stage CUDA events on subsequent calls (see include/hyde.h HYDE_STAGE_*)."""
    h = handle(device)
    check(lib().hyde_profile_enable(h, 1 if on else 0), h)


def profile_read(device: int = 0):
    """Synchronize and return {stage: (ms, kernel launches)} accumulated since the last read."""
    h = handle(device)
    ms = (ctypes.c_double * 8)()
    nl = (ctypes.c_longlong * 8)()
    check(lib().hyde_profile_read(h, ms, nl), h)
    return {name: (ms[i], nl[i]) for i, name in enumerate(_lib.STAGES)}


def launch_count(device: int = 0) -> int:
    return int(lib().hyde_launch_count(handle(device)))


def eig_cluster_size() -> int:
    """CTAs in the K2 eigensolver cluster on this device (16, or 8 when 16 cannot co-schedule)."""
    return int(lib().hyde_eig_cluster_size())
