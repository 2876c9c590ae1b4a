"""CPU-side checks of the C-ABI library: it loads, exports every function include/hyde.h
declares, and its host-side helpers (filters, level rule, coefficient count) agree with the
oracle.  No GPU compute is called here."""
import ctypes
import os

import numpy as np
import pytest

from oracle import hyres_ref as O
from paper_2204_06979_b200 import _lib
from paper_2204_06979_b200.build import LIB, build


@pytest.fixture(scope="module")
def L():
    build()
    return _lib.lib()


def test_header_symbols_exported(L):
    names = _lib.header_functions()
    assert len(names) >= 20
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing
    # and the binding declares a signature for each of them
    assert sorted(_lib._SIGS) == names


def test_library_targets_sm100a(L):
    assert L.hyde_target_sm() == 100
    assert b"sm_100a" in L.hyde_version()
    out = os.popen(f"cuobjdump --list-elf {LIB} 2>/dev/null").read()
    if out:
        assert "sm_100a" in out


@pytest.mark.parametrize("taps", [2, 8, 16])
def test_library_filters_match_oracle(L, taps):
    buf = (ctypes.c_double * taps)()
    assert L.hyde_filter(taps, buf) == 0
    h, _ = O.filters(taps)
    assert np.max(np.abs(np.array(buf[:]) - h)) < 1e-15


def test_library_filter_rejects_unknown(L):
    buf = (ctypes.c_double * 16)()
    assert L.hyde_filter(6, buf) == _lib.HYDE_EPARAM


def test_levels_and_counts_match_oracle(L):
    for r, c in [(64, 64), (145, 145), (610, 340), (349, 1905), (1024, 1024), (256, 256), (17, 33), (15, 200), (30, 31)]:
        for taps in (2, 8, 16):
            assert L.hyde_auto_levels(r, c, taps) == O.auto_levels(r, c, taps), (r, c, taps)
        for lv in range(1, 5):
            if min(r, c) >= 2 ** lv:
                assert L.hyde_dwt_coeff_count(r, c, lv) == O.coeff_count(r, c, lv)


def test_params_default(L):
    p = _lib.Params()
    L.hyde_hyres_params_default(ctypes.byref(p))
    assert (p.wavelet_taps, p.levels, p.chunk, p.ridge, p.flags) == (16, 0, 16, 1e-6, 0)
    assert L.hyde_hyres_workspace_size(1024, 1024, 224, 1, None) > 4 * 16 * 1024 * 1024


def test_status_strings(L):
    for s in (0, 2, 3, 4, 5, 6, 7):
        assert L.hyde_status_string(s)


def test_null_handle_is_param_error(L):
    assert L.hyde_hyres(None, None, 8, 8, 4, None, None) == _lib.HYDE_EPARAM
    assert L.hyde_destroy(None) == 0
