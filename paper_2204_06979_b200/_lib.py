"""ctypes binding of libhyde.so (include/hyde.h).  Argument marshalling only.

There is no fallback: if libhyde.so is missing or a call fails, this raises.
"""
from __future__ import annotations

import ctypes
import os
import re
from ctypes import POINTER, c_char_p, c_double, c_float, c_int, c_size_t, c_void_p

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG_DIR, "libhyde.so")
HEADER = os.path.join(os.path.dirname(PKG_DIR), "include", "hyde.h")

HYDE_OK, HYDE_EPARAM, HYDE_EDATA, HYDE_EMETHOD, HYDE_ECUDA, HYDE_ENCCL, HYDE_ENOMEM = 0, 2, 3, 4, 5, 6, 7
HYDE_KEEP_LL = 1
HYDE_VALIDATE = 2
STAGES = ("gram", "eig", "project", "dwt", "sure", "rank", "idwt", "recon")


class HydeError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"hyde status {status}: {msg}")
        self.status = status


class Params(ctypes.Structure):
    _fields_ = [("wavelet_taps", c_int), ("levels", c_int), ("chunk", c_int),
                ("ridge", c_double), ("flags", c_int)]


class Info(ctypes.Structure):
    _fields_ = [("rank", c_int), ("levels", c_int), ("chunks_run", c_int),
                ("nonfinite_input", c_int), ("n_coeffs", c_int), ("comps", c_int),
                ("reserved", c_int * 2)]

    def as_dict(self):
        return {"rank": self.rank, "levels": self.levels, "chunks_run": self.chunks_run,
                "nonfinite_input": self.nonfinite_input, "n_coeffs": self.n_coeffs,
                "comps": self.comps}


_P = c_void_p  # device or host pointer

# hyde_comm callbacks (include/hyde.h): device pointers, the caller's stream
ALLREDUCE_FN = ctypes.CFUNCTYPE(c_int, c_void_p, c_void_p, c_size_t, c_void_p)


class P2p(ctypes.Structure):
    _fields_ = [("peer", c_int), ("buf", c_void_p), ("bytes", c_size_t)]


SENDRECV_FN = ctypes.CFUNCTYPE(c_int, c_void_p, c_int, POINTER(P2p), c_int, POINTER(P2p), c_void_p)


class Comm(ctypes.Structure):
    _fields_ = [("rank", c_int), ("world", c_int), ("user", c_void_p),
                ("allreduce_sum_f64", ALLREDUCE_FN), ("sendrecv", SENDRECV_FN)]


_SIGS = {
    "hyde_create": (c_int, [POINTER(c_void_p), c_int]),
    "hyde_destroy": (c_int, [c_void_p]),
    "hyde_status_string": (c_char_p, [c_int]),
    "hyde_last_error": (c_char_p, [c_void_p]),
    "hyde_version": (c_char_p, []),
    "hyde_target_sm": (c_int, []),
    "hyde_hyres_params_default": (None, [POINTER(Params)]),
    "hyde_estimate_noise": (c_int, [c_void_p, _P, c_int, c_int, c_int, _P, _P, _P, c_void_p]),
    "hyde_hyres": (c_int, [c_void_p, _P, c_int, c_int, c_int, _P, c_void_p]),
    "hyde_hyres_ex": (c_int, [c_void_p, _P, c_int, c_int, c_int, _P, POINTER(Params), POINTER(Info), c_void_p]),
    "hyde_hyres_host": (c_int, [c_void_p, _P, c_int, c_int, c_int, _P, POINTER(Params), POINTER(Info), c_void_p]),
    "hyde_hyres_host_stream": (c_int, [c_void_p, POINTER(c_void_p), POINTER(c_void_p), c_int, c_int, c_int, c_int,
                                       POINTER(Params), POINTER(Info), c_void_p]),
    "hyde_hyres_sharded": (c_int, [c_void_p, c_void_p, _P, c_int, c_int, c_int, c_int, c_int, _P, POINTER(Params),
                                   POINTER(Info), c_void_p]),
    "hyde_hyres_sharded_cb": (c_int, [c_void_p, POINTER(Comm), _P, c_int, c_int, c_int, c_int, c_int, _P,
                                      POINTER(Params), POINTER(Info), c_void_p]),
    "hyde_nccl_version": (c_int, []),
    "hyde_nccl_unique_id": (c_int, [c_void_p]),
    "hyde_nccl_comm_init": (c_int, [POINTER(c_void_p), c_int, c_int, c_void_p, c_int]),
    "hyde_nccl_comm_destroy": (c_int, [c_void_p]),
    "hyde_shard_rows": (c_int, [c_int, c_int, c_int, POINTER(c_int), POINTER(c_int)]),
    "hyde_shard_owner": (c_int, [c_int, c_int]),
    "hyde_hyres_workspace_size": (c_size_t, [c_int, c_int, c_int, c_int, POINTER(Params)]),
    "hyde_hyres_batched": (c_int, [c_void_p, _P, c_int, c_int, c_int, c_int, _P, POINTER(Params), POINTER(Info), c_void_p]),
    "hyde_sync_status": (c_int, [c_void_p, c_void_p]),
    "hyde_l1_spectral": (c_int, [c_void_p, _P, c_int, c_int, c_int, _P, c_double, c_double, c_int, c_double, _P,
                                 c_void_p]),
    "hyde_hyminor": (c_int, [c_void_p, _P, c_int, c_int, c_int, _P, c_double, c_double, c_int, c_double, POINTER(Info),
                             c_void_p]),
    "hyde_wsrrr": (c_int, [c_void_p, _P, c_int, c_int, c_int, c_int, c_double, c_int, c_int, c_int, c_double, _P, _P,
                           POINTER(c_int), POINTER(c_double), POINTER(c_int), POINTER(c_double), c_void_p]),
    "hyde_forpdn": (c_int, [c_void_p, _P, c_int, c_int, c_int, _P, c_double, c_int, c_int, POINTER(c_double),
                            c_void_p]),
    "hyde_hysime": (c_int, [c_void_p, _P, c_int, c_int, c_int, POINTER(c_int), _P, _P, _P, _P, c_void_p]),
    "hyde_k_gram": (c_int, [c_void_p, _P, c_int, c_int, _P, c_void_p]),
    "hyde_k_eig": (c_int, [c_void_p, _P, c_int, c_int, c_double, c_int, _P, _P, _P, c_void_p]),
    "hyde_k_project": (c_int, [c_void_p, _P, c_int, c_int, _P, c_int, _P, c_void_p]),
    "hyde_k_dwt_fwd": (c_int, [c_void_p, _P, c_int, c_int, c_int, c_int, c_int, _P, c_void_p]),
    "hyde_dwt_coeff_count": (c_int, [c_int, c_int, c_int]),
    "hyde_auto_levels": (c_int, [c_int, c_int, c_int]),
    "hyde_k_sure": (c_int, [c_void_p, _P, c_int, c_int, c_int, c_int, c_int, _P, _P, _P, c_void_p]),
    "hyde_k_idwt": (c_int, [c_void_p, _P, c_int, c_int, c_int, c_int, c_int, _P, c_void_p]),
    "hyde_wavelet_shrink": (c_int, [c_void_p, _P, c_int, c_int, c_int, c_int, c_int, c_int, _P, _P, _P, _P,
                                    c_void_p]),
    "hyde_k_reconstruct": (c_int, [c_void_p, _P, c_int, c_int, _P, c_int, c_int, _P, c_void_p]),
    "hyde_filter": (c_int, [c_int, POINTER(c_double)]),
    "hyde_profile_enable": (c_int, [c_void_p, c_int]),
    "hyde_profile_read": (c_int, [c_void_p, POINTER(c_double), POINTER(ctypes.c_longlong)]),
    "hyde_launch_count": (ctypes.c_longlong, [c_void_p]),
    "hyde_debug_eig_clocks": (c_int, [POINTER(ctypes.c_longlong)]),
    "hyde_debug_eig_lanczos": (c_int, [c_int, c_int]),
    "hyde_eig_cluster_size": (c_int, []),
    "hyde_debug_sure_prof": (c_int, [POINTER(ctypes.c_ulonglong)]),
    "hyde_debug_eig_state": (c_int, [c_void_p, c_int, c_int, _P, _P]),
    "hyde_debug_gram_quant": (c_int, [c_void_p, c_int, c_int, _P, _P, _P]),
}

_lib = None


def header_functions(path: str = HEADER):
    """Names of the functions include/hyde.h declares."""
    txt = open(path).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(hyde_[a-z0-9_]+)\s*\(", txt)))


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise HydeError(-1, f"{LIB_PATH} is not built: run `python -m paper_2204_06979_b200.build`")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(status: int, handle=None):
    if status != HYDE_OK:
        msg = lib().hyde_last_error(handle).decode(errors="replace")
        raise HydeError(status, msg)


def make_params(taps=16, levels=0, chunk=16, ridge=1e-6, keep_ll=False, validate=False) -> Params:
    p = Params()
    lib().hyde_hyres_params_default(ctypes.byref(p))
    p.wavelet_taps = int(taps)
    p.levels = int(levels)
    p.chunk = int(chunk)
    p.ridge = float(ridge)
    p.flags = (HYDE_KEEP_LL if keep_ll else 0) | (HYDE_VALIDATE if validate else 0)
    return p
