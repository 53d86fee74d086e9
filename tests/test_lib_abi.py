"""C-ABI library checks that need no GPU (-m "not gpu").

* libkkrx.so loads and exports every function declared in include/kk_rx.h
* the C++ built-in constellations equal the committed data files (which the
  oracle pins), i.e. both sides see the same points and labels
* argument validation fails with KK_EINVAL before touching CUDA
* halo geometry covers what the method needs (oracle.required_left/right)
"""
import ctypes as C
import os
import re

import numpy as np
import pytest

from paper_2108_07004_b200 import _lib
from paper_2108_07004_b200.receiver import builtin_constellation, halo_for


def _declared_functions(root):
    txt = open(os.path.join(root, "include", "kk_rx.h")).read()
    return sorted(set(re.findall(r"^\s*(?:[a-z_0-9]+\s*\*?\s*)+?\b(kk_rx_[a-z_0-9]+)\s*\(", txt, re.M)))


def test_library_exports_every_declared_symbol(root):
    lib = _lib.load()
    names = _declared_functions(root)
    assert len(names) >= 15
    for n in names:
        assert hasattr(lib, n), n
        assert n in _lib.EXPORTS, f"binding misses {n}"
    assert lib.kk_rx_abi_version() == 2


def test_builtin_constellations_match_data_files(root):
    from synth.generate import load_constellation
    for fmt in ("QAM4", "QAM8", "QAM16", "QAM32", "QAM64", "QAM128"):
        p, l = builtin_constellation(fmt)
        q, lq = load_constellation(fmt)
        assert np.max(np.abs(p - q)) < 1e-6 and np.array_equal(l, lq)
    with pytest.raises(ValueError):
        builtin_constellation("GS8")


def test_params_default_and_validation():
    lib = _lib.load()
    p = _lib.KKParams()
    lib.kk_rx_params_default(C.byref(p))
    assert p.tone_bin == 541065 and p.k_update == 4096 and abs(p.mu - 1e-3) < 1e-9 and p.fir_len == 203
    h = C.c_void_p()
    # no fir -> EINVAL
    assert lib.kk_rx_create(C.byref(h), 0, 4, 1 << 22, 12.0, C.byref(p)) == _lib.KK_EINVAL
    fir = np.zeros(406, np.float32)
    p.fir = fir.ctypes.data_as(C.POINTER(C.c_float))
    p.dc_offset = 1000.0
    assert lib.kk_rx_create(C.byref(h), 0, 2, 1 << 22, 12.0, C.byref(p)) == _lib.KK_EINVAL       # sps
    assert lib.kk_rx_create(C.byref(h), 0, 4, (1 << 22) + 100, 12.0, C.byref(p)) == _lib.KK_EINVAL  # N % 512
    assert lib.kk_rx_create(C.byref(h), 6, 4, 1 << 22, 12.0, C.byref(p)) == _lib.KK_EINVAL       # GS8 w/o points
    p.sub_block = 3
    assert lib.kk_rx_create(C.byref(h), 0, 4, 1 << 22, 12.0, C.byref(p)) == _lib.KK_EINVAL       # L does not divide
    p.sub_block = 0
    p.update_mode = 1
    assert lib.kk_rx_create(C.byref(h), 0, 4, 1 << 22, 12.0, C.byref(p)) == _lib.KK_EINVAL       # PILOT w/o pattern
    assert b"PILOT" in lib.kk_rx_last_error(None)
    assert lib.kk_rx_destroy(None) == _lib.KK_OK


def test_halo_covers_method_needs():
    from oracle import kk_oracle as O
    for n in (1 << 16, 1 << 22, 66048):
        left, right = halo_for(n, 4096)
        assert left >= O.required_left(4096) and right >= O.required_right()
    assert halo_for(1 << 22, 4096) == (17672, 2312)


def test_cufft_comparison_library_exports(root):
    """libkkrx_cufft.so (the cuFFT comparison pipeline, never the product path) loads,
    exports what include/kk_cufft_cmp.h declares, and validates its arguments without CUDA."""
    from paper_2108_07004_b200 import cufft_cmp
    lib = cufft_cmp.load()
    txt = open(os.path.join(root, "include", "kk_cufft_cmp.h")).read()
    names = sorted(set(re.findall(r"^\s*int\s+(kk_cmp_[a-z_0-9]+)\s*\(", txt, re.M)))
    assert len(names) == 5 and tuple(names) == tuple(sorted(cufft_cmp.EXPORTS))
    for n in names:
        assert hasattr(lib, n), n
    h = C.c_void_p()
    fir = np.zeros(406, np.float32)
    fp = fir.ctypes.data_as(C.POINTER(C.c_float))
    assert lib.kk_cmp_create(C.byref(h), (1 << 16) + 512, 1, 1000.0, 10.0, 1.0, 541065, fp, 203) == -1  # N % 1024
    assert lib.kk_cmp_create(C.byref(h), 1 << 16, 1, 1000.0, 10.0, 1.0, 541065, fp, 202) == -1         # fir_len
    assert lib.kk_cmp_create(C.byref(h), 1 << 16, 0, 1000.0, 10.0, 1.0, 541065, fp, 203) == -1         # batch
    assert lib.kk_cmp_destroy(None) == 0


def test_new_entry_points_reject_bad_arguments():
    """The sweep / CSPR / frame-sync / training calls validate their arguments before any
    CUDA work (KK_EINVAL with a NULL handle or impossible sizes; no GPU needed)."""
    lib = _lib.load()
    f = np.ones(4, np.float32)
    fp = f.ctypes.data_as(C.POINTER(C.c_float))
    cnt = (_lib.KKCounts * 4)()
    best = C.c_int()
    k = C.c_int64()
    assert lib.kk_rx_set_cspr(None, 12.0) == _lib.KK_EINVAL
    assert lib.kk_rx_sweep(None, None, 1, fp, None, 4, cnt, C.byref(best)) == _lib.KK_EINVAL
    assert lib.kk_rx_dc_sweep(None, None, 1, fp, 4, cnt, C.byref(best)) == _lib.KK_EINVAL
    assert lib.kk_rx_frame_sync(None, None, 0, 2048, C.byref(k), None, None) == _lib.KK_EINVAL
    assert lib.kk_rx_train_fir(None, None, fp, 32, 2, 0.0, fp) == _lib.KK_EINVAL
    assert lib.kk_rx_train_taps(None, None, 16, fp) == _lib.KK_EINVAL
    assert lib.kk_rx_set_dc_offset(None, 100.0) == _lib.KK_EINVAL
    assert lib.kk_rx_last_error(None)
