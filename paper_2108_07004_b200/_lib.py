"""ctypes declarations of include/kk_rx.h (argument marshalling only).

The shared library is built in-tree (paper_2108_07004_b200/libkkrx.so) by
paper_2108_07004_b200.build / __graft_entry__.build().  There is no fallback:
if the library is missing, importing the binding raises.
"""
import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libkkrx.so")
# A/B measurements of kernel variants (tools/gpu/ab.sh): another in-tree build of the same library
if os.environ.get("KKRX_LIB"):
    LIB_PATH = os.path.abspath(os.environ["KKRX_LIB"])

KK_OK, KK_EINVAL, KK_ENOMEM, KK_ECUDA, KK_ESTATE, KK_EUNSUPPORTED = 0, -1, -2, -3, -4, -5
FORMATS = {"QAM4": 0, "QAM8": 1, "QAM16": 2, "QAM32": 3, "QAM64": 4, "QAM128": 5, "GS8": 6, "GS128": 7,
           "CUSTOM": 8}
UPD_DD_SOFT, UPD_PILOT, UPD_DD_HARD = 0, 1, 2
DUMP_ES = 1


class KKParams(C.Structure):
    _fields_ = [
        ("dc_offset", C.c_float),
        ("tone_bin", C.c_int64),
        ("fir", C.POINTER(C.c_float)),
        ("fir_len", C.c_int32),
        ("w_init", C.POINTER(C.c_float)),
        ("mu", C.c_float),
        ("k_update", C.c_int32),
        ("sub_block", C.c_int32),
        ("gate_tau", C.c_float),
        ("update_mode", C.c_int32),
        ("points", C.POINTER(C.c_float)),
        ("labels", C.POINTER(C.c_uint8)),
        ("m", C.c_int32),
        ("ref_pattern", C.POINTER(C.c_uint8)),
        ("ref_len", C.c_int32),
        ("ref_offset", C.c_int64),
        ("v_min", C.c_float),
        ("device", C.c_int32),
        ("cuda_stream", C.c_void_p),
        ("debug_dump", C.c_uint32),
        ("max_batch", C.c_int32),
        ("pre_fir", C.POINTER(C.c_float)),
        ("pre_fir_len", C.c_int32),
    ]


class KKCounts(C.Structure):
    _fields_ = [
        ("bit_errors", C.c_uint64),
        ("sym_errors", C.c_uint64),
        ("bits", C.c_uint64),
        ("symbols", C.c_uint64),
        ("clipped_samples", C.c_uint64),
        ("gated_updates", C.c_uint64),
        ("flags", C.c_uint32),
        ("reserved", C.c_uint32),
    ]

    def as_dict(self):
        return {f: int(getattr(self, f)) for f, _ in self._fields_ if f != "reserved"}


# numpy view of kk_rx_counts (same layout): bulk counters without per-buffer Python objects
COUNTS_DTYPE = np.dtype([("bit_errors", "<u8"), ("sym_errors", "<u8"), ("bits", "<u8"), ("symbols", "<u8"),
                         ("clipped_samples", "<u8"), ("gated_updates", "<u8"), ("flags", "<u4"), ("reserved", "<u4")])
assert COUNTS_DTYPE.itemsize == C.sizeof(KKCounts)

EXPORTS = {
    "kk_rx_params_default": (None, [C.POINTER(KKParams)]),
    "kk_rx_create": (C.c_int, [C.POINTER(C.c_void_p), C.c_int, C.c_int, C.c_int64, C.c_float, C.POINTER(KKParams)]),
    "kk_rx_halo": (C.c_int, [C.c_void_p, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "kk_rx_halo_for": (C.c_int, [C.c_int64, C.c_int32, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "kk_rx_process": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(KKCounts)]),
    "kk_rx_process_batch": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.POINTER(KKCounts)]),
    "kk_rx_seek": (C.c_int, [C.c_void_p, C.c_int64]),
    "kk_rx_submit_batch": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]),
    "kk_rx_submit_batch_packed12": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]),
    "kk_rx_sync": (C.c_int, [C.c_void_p, C.POINTER(KKCounts), C.c_int64, C.POINTER(C.c_int64)]),
    "kk_rx_async_launches": (C.c_int64, [C.c_void_p]),
    "kk_rx_pageable_staged": (C.c_int, [C.c_void_p, C.POINTER(C.c_int64)]),
    "kk_rx_set_dc_offset": (C.c_int, [C.c_void_p, C.c_float]),
    "kk_gmi_awgn": (C.c_int, [C.POINTER(C.c_float), C.POINTER(C.c_uint8), C.c_int, C.c_int, C.c_double, C.c_int,
                              C.POINTER(C.c_double)]),
    "kk_hermgauss": (C.c_int, [C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "kk_rx_train_fir": (C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(C.c_float), C.c_int64, C.c_int64, C.c_double,
                                  C.POINTER(C.c_float)]),
    "kk_rx_set_fir": (C.c_int, [C.c_void_p, C.POINTER(C.c_float)]),
    "kk_rx_train_taps": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.POINTER(C.c_float)]),
    "kk_rx_frame_sync": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.POINTER(C.c_int64),
                                   C.POINTER(C.c_float), C.POINTER(C.c_double)]),
    "kk_rx_set_w_init": (C.c_int, [C.c_void_p, C.POINTER(C.c_float)]),
    "kk_rx_dc_sweep": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.POINTER(C.c_float), C.c_int,
                                 C.POINTER(KKCounts), C.POINTER(C.c_int)]),
    "kk_rx_sweep": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.POINTER(C.c_float), C.POINTER(C.c_float), C.c_int,
                              C.POINTER(KKCounts), C.POINTER(C.c_int)]),
    "kk_rx_set_cspr": (C.c_int, [C.c_void_p, C.c_float]),
    "kk_rx_get_taps": (C.c_int, [C.c_void_p, C.c_int64, C.POINTER(C.c_float)]),
    "kk_rx_totals": (C.c_int, [C.c_void_p, C.POINTER(KKCounts)]),
    "kk_rx_reset_totals": (C.c_int, [C.c_void_p]),
    "kk_rx_debug_x2": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64, C.POINTER(C.c_float)]),
    "kk_rx_debug_es": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64, C.POINTER(C.c_float)]),
    "kk_rx_constellation": (C.c_int, [C.c_int, C.POINTER(C.c_float), C.POINTER(C.c_uint8)]),
    "kk_rx_last_launches": (C.c_int64, [C.c_void_p]),
    "kk_rx_decision_tables": (C.c_int, [C.POINTER(C.c_float), C.c_int, C.c_float, C.POINTER(C.c_float),
                                        C.POINTER(C.c_float), C.POINTER(C.c_uint32), C.POINTER(C.c_float)]),
    "kk_rx_set_timing": (C.c_int, [C.c_void_p, C.c_int]),
    "kk_rx_kernel_times": (C.c_int, [C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_int64)]),
    "kk_rx_last_error": (C.c_char_p, [C.c_void_p]),
    "kk_rx_destroy": (C.c_int, [C.c_void_p]),
    "kk_rx_abi_version": (C.c_int, []),
}

_lib = None


def load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() (no CPU fallback exists)")
        lib = C.CDLL(LIB_PATH)
        for name, (res, args) in EXPORTS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


class KKError(RuntimeError):
    pass


def check(status, what=""):
    if status != KK_OK:
        msg = load().kk_rx_last_error(None)
        raise KKError(f"{what} failed with status {status}: {msg.decode() if msg else ''}")
