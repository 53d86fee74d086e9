"""ctypes binding of include/kk_cufft_cmp.h: the cuFFT multi-kernel S1-S4 pipeline.

COMPARISON ONLY (north star: cuFFT "reported only as a comparison").
bench.py times it beside the fused chain; tests/test_gpu_parity.py checks its x2 against
the oracle.  Nothing in the product path (receiver.py, libkkrx.so) uses it.
"""
import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libkkrx_cufft.so")
_lib = None


def load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run paper_2108_07004_b200.build.build_cmp()")
        L = C.CDLL(LIB_PATH)
        L.kk_cmp_create.argtypes = [C.POINTER(C.c_void_p), C.c_int64, C.c_int, C.c_float, C.c_float, C.c_float,
                                    C.c_int64, C.POINTER(C.c_float), C.c_int]
        L.kk_cmp_halo.argtypes = [C.c_void_p, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
        L.kk_cmp_x2.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p]
        L.kk_cmp_launches.argtypes = [C.c_void_p, C.c_int]
        L.kk_cmp_destroy.argtypes = [C.c_void_p]
        for f in ("kk_cmp_create", "kk_cmp_halo", "kk_cmp_x2", "kk_cmp_launches", "kk_cmp_destroy"):
            getattr(L, f).restype = C.c_int
        _lib = L
    return _lib


EXPORTS = ("kk_cmp_create", "kk_cmp_halo", "kk_cmp_x2", "kk_cmp_launches", "kk_cmp_destroy")


class CufftS1S4:
    """x2 of whole buffers through cuFFT (see the header for the stage list)."""

    def __init__(self, buffer_len, max_batch, dc_offset, cspr_db, fir, tone_bin=541065, v_min=1.0):
        L = load()
        c = 10.0 ** (cspr_db / 10.0)
        a_hat = float(np.sqrt(np.float64(np.float32(dc_offset)) * c / (1.0 + c)))  # reading R6
        f = np.ascontiguousarray(np.stack([np.real(fir), np.imag(fir)], 1).astype(np.float32).ravel())
        self.h = C.c_void_p()
        rc = L.kk_cmp_create(C.byref(self.h), int(buffer_len), int(max_batch), float(dc_offset), a_hat, float(v_min),
                             int(tone_bin), f.ctypes.data_as(C.POINTER(C.c_float)), len(fir))
        if rc != 0:
            raise RuntimeError(f"kk_cmp_create failed ({rc})")
        self.buffer_len = buffer_len
        self.L = L

    def halo(self):
        a, b = C.c_int64(), C.c_int64()
        self.L.kk_cmp_halo(self.h, C.byref(a), C.byref(b))
        return a.value, b.value

    def x2(self, codes, first, nbuf, out, stream=0):
        """codes: cuda int16 tensor (a stream); first: index of buffer 0's first sample;
        out: cuda complex64 tensor of nbuf * buffer_len / 2 (enqueued, not synchronised)."""
        rc = self.L.kk_cmp_x2(self.h, codes.data_ptr() + 2 * int(first), int(nbuf), out.data_ptr(), C.c_void_p(stream))
        if rc != 0:
            raise RuntimeError(f"kk_cmp_x2 failed ({rc})")

    def launches(self, nbuf):
        return self.L.kk_cmp_launches(self.h, int(nbuf))

    def close(self):
        if self.h:
            self.L.kk_cmp_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
