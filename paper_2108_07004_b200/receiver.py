"""Thin Python binding of the kk_rx C ABI (same names; marshalling only).

Every step of the receiver runs in libkkrx.so's sm_100a kernels; this module
only converts Python/NumPy/torch arguments into the C structs and pointers of
include/kk_rx.h.  torch is used for device memory and streams only.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from ._lib import COUNTS_DTYPE, KKCounts, KKParams, check


def _ptr(obj):
    """Raw address of a torch tensor or NumPy array (no copies)."""
    if hasattr(obj, "data_ptr"):
        return obj.data_ptr(), obj.element_size()
    if isinstance(obj, np.ndarray):
        assert obj.flags["C_CONTIGUOUS"]
        return obj.ctypes.data, obj.itemsize
    raise TypeError(type(obj))


def _fptr(a):
    return a.ctypes.data_as(C.POINTER(C.c_float))


def _u8ptr(a):
    return a.ctypes.data_as(C.POINTER(C.c_uint8))


class KKReceiver:
    """kk_rx_create / kk_rx_process(_batch) / kk_rx_destroy."""

    def __init__(self, fmt, buffer_len, cspr_db, fir, dc_offset, *, points=None, labels=None, tone_bin=541065,
                 w_init=None, mu=1e-3, k_update=4096, sub_block=0, gate_tau=-1.0, update_mode=0, ref_pattern=None,
                 ref_offset=0, v_min=1.0, device=-1, stream=None, debug_dump=0, max_batch=16, pre_fir=None):
        lib = _lib.load()
        self._lib = lib
        p = KKParams()
        lib.kk_rx_params_default(C.byref(p))
        self._keep = []
        fir = np.asarray(fir, dtype=np.complex128)
        fir_f = np.ascontiguousarray(np.stack([fir.real, fir.imag], -1).reshape(-1).astype(np.float32))
        self._keep.append(fir_f)
        p.fir = _fptr(fir_f)
        p.fir_len = len(fir)
        p.dc_offset = float(np.float32(dc_offset))
        p.tone_bin = int(tone_bin)
        if w_init is not None:
            w = np.asarray(w_init, dtype=np.complex128).reshape(8)
            wf = np.ascontiguousarray(np.stack([w.real, w.imag], -1).reshape(-1).astype(np.float32))
            self._keep.append(wf)
            p.w_init = _fptr(wf)
        p.mu = mu
        p.k_update = k_update
        p.sub_block = sub_block
        p.gate_tau = gate_tau
        p.update_mode = update_mode
        if points is not None:
            pts = np.asarray(points, dtype=np.complex128)
            pf = np.ascontiguousarray(np.stack([pts.real, pts.imag], -1).reshape(-1).astype(np.float32))
            lb = np.ascontiguousarray(np.asarray(labels, dtype=np.uint8))
            self._keep += [pf, lb]
            p.points = _fptr(pf)
            p.labels = _u8ptr(lb)
            p.m = len(pts)
        if ref_pattern is not None:
            rp = np.ascontiguousarray(np.asarray(ref_pattern, dtype=np.uint8))
            self._keep.append(rp)
            p.ref_pattern = _u8ptr(rp)
            p.ref_len = len(rp)
        p.ref_offset = int(ref_offset)
        p.v_min = v_min
        p.device = device
        p.cuda_stream = stream
        p.debug_dump = debug_dump
        p.max_batch = max_batch
        if pre_fir is not None:
            pf = np.ascontiguousarray(np.asarray(pre_fir, dtype=np.float32))
            self._keep.append(pf)
            p.pre_fir = _fptr(pf)
            p.pre_fir_len = len(pf)
        fmt_id = _lib.FORMATS[fmt] if isinstance(fmt, str) else int(fmt)
        h = C.c_void_p()
        check(lib.kk_rx_create(C.byref(h), fmt_id, 4, int(buffer_len), float(cspr_db), C.byref(p)), "kk_rx_create")
        self.h = h
        self.buffer_len = int(buffer_len)
        self.n_sym = self.buffer_len // 4
        self.nsub = self.n_sym // (sub_block if sub_block > 0 else self.n_sym)
        self.max_batch = max_batch

    # ------------------------------------------------------------------
    def halo(self):
        l, r = C.c_int64(), C.c_int64()
        check(self._lib.kk_rx_halo(self.h, C.byref(l), C.byref(r)), "kk_rx_halo")
        return l.value, r.value

    def seek(self, buffer_index):
        check(self._lib.kk_rx_seek(self.h, int(buffer_index)), "kk_rx_seek")

    def process_batch(self, stream, offset, nbuf, out=None, as_array=False):
        """stream: int16 torch tensor (cuda or pinned cpu) or NumPy array holding
        the contiguous sample stream; offset: index of buffer 0's first sample.
        out: uint8 tensor/array of nbuf*N/4 labels or None.  Returns a list of
        per-buffer counter dicts."""
        base, es = _ptr(stream)
        assert es == 2
        optr = None
        if out is not None:
            optr, _ = _ptr(out)
        buf = self._counts_buf(nbuf)
        check(self._lib.kk_rx_process_batch(self.h, C.c_void_p(base + 2 * int(offset)), int(nbuf),
                                            C.c_void_p(optr) if optr is not None else None,
                                            buf.ctypes.data_as(C.POINTER(KKCounts))), "kk_rx_process_batch")
        arr = buf[:int(nbuf)].copy()
        return arr if as_array else self._as_dicts(arr)

    def submit_batch(self, stream, offset, nbuf, out=None):
        """Asynchronous kk_rx_submit_batch: enqueue nbuf buffers (see process_batch for
        the arguments); outputs and counters become valid at sync()."""
        base, es = _ptr(stream)
        assert es == 2
        optr = None
        if out is not None:
            optr, _ = _ptr(out)
        check(self._lib.kk_rx_submit_batch(self.h, C.c_void_p(base + 2 * int(offset)), int(nbuf),
                                           C.c_void_p(optr) if optr is not None else None), "kk_rx_submit_batch")

    def submit_batch_packed12(self, packed, offset, nbuf, out=None):
        """kk_rx_submit_batch_packed12: `packed` holds the stream in the packed 12-bit
        format (uint8, 3 bytes per 2 samples; host or device); offset = sample index of
        buffer 0's first sample (even)."""
        base, es = _ptr(packed)
        assert es == 1 and int(offset) % 2 == 0
        optr = None
        if out is not None:
            optr, _ = _ptr(out)
        check(self._lib.kk_rx_submit_batch_packed12(self.h, C.c_void_p(base + 3 * int(offset) // 2), int(nbuf),
                                                    C.c_void_p(optr) if optr is not None else None),
              "kk_rx_submit_batch_packed12")

    def _counts_buf(self, n):
        if getattr(self, "_cbuf", None) is None or len(self._cbuf) < n:
            self._cbuf = np.zeros(max(int(n), 1), dtype=COUNTS_DTYPE)
        return self._cbuf

    @staticmethod
    def _as_dicts(arr):
        names = [f for f in COUNTS_DTYPE.names if f != "reserved"]
        return [{f: int(r[f]) for f in names} for r in arr]

    def sync(self, max_out=1 << 16, as_array=False):
        """kk_rx_sync: wait for every submitted batch; per-buffer counters in order, as dicts
        or (as_array) one numpy structured array (COUNTS_DTYPE, no per-buffer objects)."""
        buf = self._counts_buf(max_out)
        n = C.c_int64()
        check(self._lib.kk_rx_sync(self.h, buf.ctypes.data_as(C.POINTER(KKCounts)), int(max_out), C.byref(n)),
              "kk_rx_sync")
        arr = buf[:min(n.value, max_out)].copy()
        return arr if as_array else self._as_dicts(arr)

    def set_dc_offset(self, dc_offset):
        check(self._lib.kk_rx_set_dc_offset(self.h, float(dc_offset)), "kk_rx_set_dc_offset")

    def dc_sweep(self, stream, offset, nbuf, dc_values):
        """kk_rx_dc_sweep: counters (summed over the nbuf buffers) per DC offset and the
        index of the best (lowest BER) offset."""
        base, es = _ptr(stream)
        assert es == 2
        dv = np.ascontiguousarray(np.asarray(dc_values, dtype=np.float32))
        cnt = (KKCounts * len(dv))()
        best = C.c_int()
        check(self._lib.kk_rx_dc_sweep(self.h, C.c_void_p(base + 2 * int(offset)), int(nbuf), _fptr(dv), len(dv),
                                       cnt, C.byref(best)), "kk_rx_dc_sweep")
        return [c.as_dict() for c in cnt], int(best.value)

    def set_cspr(self, cspr_db):
        check(self._lib.kk_rx_set_cspr(self.h, float(cspr_db)), "kk_rx_set_cspr")

    def sweep(self, stream, offset, nbuf, dc_values, cspr_db_values=None):
        """kk_rx_sweep: counters (summed over the nbuf buffers) per (DC offset, CSPR)
        hypothesis and the index of the best (lowest BER) one."""
        base, es = _ptr(stream)
        assert es == 2
        dv = np.ascontiguousarray(np.asarray(dc_values, dtype=np.float32))
        cv = None if cspr_db_values is None else np.ascontiguousarray(np.asarray(cspr_db_values, dtype=np.float32))
        assert cv is None or len(cv) == len(dv)
        cnt = (KKCounts * len(dv))()
        best = C.c_int()
        check(self._lib.kk_rx_sweep(self.h, C.c_void_p(base + 2 * int(offset)), int(nbuf), _fptr(dv),
                                    _fptr(cv) if cv is not None else None, len(dv), cnt, C.byref(best)),
              "kk_rx_sweep")
        return [c.as_dict() for c in cnt], int(best.value)

    def train_fir(self, stream, offset, symbols, n_first, ridge=1e-9):
        """kk_rx_train_fir: LS 203-tap static equaliser from the buffer at `offset` whose
        transmitted symbols n_first .. n_first+len(symbols)-1 are `symbols` (complex)."""
        base, es = _ptr(stream)
        assert es == 2
        sy = np.asarray(symbols, dtype=np.complex128)
        sf = np.ascontiguousarray(np.stack([sy.real, sy.imag], -1).reshape(-1).astype(np.float32))
        out = np.empty(406, dtype=np.float32)
        check(self._lib.kk_rx_train_fir(self.h, C.c_void_p(base + 2 * int(offset)), _fptr(sf), int(n_first), len(sy),
                                        float(ridge), _fptr(out)), "kk_rx_train_fir")
        return out[0::2] + 1j * out[1::2].astype(np.float64)

    def set_fir(self, fir):
        f = np.asarray(fir, dtype=np.complex128)
        ff = np.ascontiguousarray(np.stack([f.real, f.imag], -1).reshape(-1).astype(np.float32))
        check(self._lib.kk_rx_set_fir(self.h, _fptr(ff)), "kk_rx_set_fir")

    def train_taps(self, stream, offset, k_steps):
        """kk_rx_train_taps: (w[4], g[4]) after k_steps PILOT LMS steps on the buffer at `offset`."""
        base, es = _ptr(stream)
        assert es == 2
        out = np.empty(16, dtype=np.float32)
        check(self._lib.kk_rx_train_taps(self.h, C.c_void_p(base + 2 * int(offset)), int(k_steps), _fptr(out)),
              "kk_rx_train_taps")
        c = out[0::2] + 1j * out[1::2].astype(np.float64)
        return c[:4], c[4:]

    def frame_sync(self, stream, offset, n0=64, n_corr=2048):
        """kk_rx_frame_sync: (n_off, c(n_off) complex, peak-to-mean ratio) of the buffer at
        `offset`: the symbol sent at buffer index n is pattern[(n + n_off) mod P]."""
        base, es = _ptr(stream)
        assert es == 2
        k = C.c_int64()
        pk = np.zeros(2, dtype=np.float32)
        ratio = C.c_double()
        check(self._lib.kk_rx_frame_sync(self.h, C.c_void_p(base + 2 * int(offset)), int(n0), int(n_corr), C.byref(k),
                                          _fptr(pk), C.byref(ratio)), "kk_rx_frame_sync")
        return int(k.value), complex(pk[0], pk[1]), float(ratio.value)

    def set_w_init(self, w, g):
        c = np.r_[np.asarray(w, dtype=np.complex128), np.asarray(g, dtype=np.complex128)]
        ff = np.ascontiguousarray(np.stack([c.real, c.imag], -1).reshape(-1).astype(np.float32))
        check(self._lib.kk_rx_set_w_init(self.h, _fptr(ff)), "kk_rx_set_w_init")

    def async_launches(self):
        return int(self._lib.kk_rx_async_launches(self.h))

    def pageable_staged(self):
        """kk_rx_pageable_staged: submissions whose pageable host input went through pinned staging."""
        n = C.c_int64(0)
        check(self._lib.kk_rx_pageable_staged(self.h, C.byref(n)), "kk_rx_pageable_staged")
        return int(n.value)

    def process(self, stream, offset, out=None):
        return self.process_batch(stream, offset, 1, out)[0]

    def taps(self, buf=0):
        a = np.empty(self.nsub * 16, dtype=np.float32)
        check(self._lib.kk_rx_get_taps(self.h, int(buf), _fptr(a)), "kk_rx_get_taps")
        c = a.reshape(self.nsub, 8, 2)
        return c[..., 0] + 1j * c[..., 1]

    def totals(self):
        c = KKCounts()
        check(self._lib.kk_rx_totals(self.h, C.byref(c)), "kk_rx_totals")
        return c.as_dict()

    def reset_totals(self):
        check(self._lib.kk_rx_reset_totals(self.h), "kk_rx_reset_totals")

    def debug_x2(self, first, count):
        a = np.empty(2 * count, dtype=np.float32)
        check(self._lib.kk_rx_debug_x2(self.h, int(first), int(count), _fptr(a)), "kk_rx_debug_x2")
        return a[0::2] + 1j * a[1::2].astype(np.float64)

    def debug_es(self, first, count):
        a = np.empty(2 * count, dtype=np.float32)
        check(self._lib.kk_rx_debug_es(self.h, int(first), int(count), _fptr(a)), "kk_rx_debug_es")
        return a[0::2] + 1j * a[1::2].astype(np.float64)

    def last_launches(self):
        return int(self._lib.kk_rx_last_launches(self.h))

    def set_timing(self, on=True):
        check(self._lib.kk_rx_set_timing(self.h, 1 if on else 0), "kk_rx_set_timing")

    def kernel_times(self):
        ms = (C.c_double * 3)()
        n = (C.c_int64 * 3)()
        check(self._lib.kk_rx_kernel_times(self.h, ms, n), "kk_rx_kernel_times")
        return {k: (ms[i], n[i]) for i, k in enumerate(("x2_pass", "lms", "chain"))}

    def close(self):
        if getattr(self, "h", None):
            self._lib.kk_rx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


def builtin_constellation(fmt):
    lib = _lib.load()
    pts = np.empty(256, dtype=np.float32)
    lab = np.empty(128, dtype=np.uint8)
    m = lib.kk_rx_constellation(_lib.FORMATS[fmt], _fptr(pts), _u8ptr(lab))
    if m < 0:
        raise ValueError(fmt)
    return pts[0:2 * m:2] + 1j * pts[1:2 * m:2].astype(np.float64), lab[:m].astype(np.int64)


def gmi_awgn(points, labels, snr_db, order=10):
    """kk_gmi_awgn: GMI (bits/symbol) of one constellation, or of a batch when points is
    [n_cand, m] and labels [n_cand, m]; returns a float or an array."""
    lib = _lib.load()
    pts = np.asarray(points, dtype=np.complex128)
    single = pts.ndim == 1
    pts = pts.reshape(-1, pts.shape[-1])
    lab = np.ascontiguousarray(np.asarray(labels, dtype=np.uint8).reshape(pts.shape))
    pf = np.ascontiguousarray(np.stack([pts.real, pts.imag], -1).reshape(-1).astype(np.float32))
    out = np.empty(pts.shape[0], dtype=np.float64)
    check(lib.kk_gmi_awgn(_fptr(pf), _u8ptr(lab), pts.shape[1], pts.shape[0], float(snr_db), int(order),
                          out.ctypes.data_as(C.POINTER(C.c_double))), "kk_gmi_awgn")
    return float(out[0]) if single else out


def hermgauss(order):
    lib = _lib.load()
    t = np.empty(order, dtype=np.float64)
    w = np.empty(order, dtype=np.float64)
    if lib.kk_hermgauss(int(order), t.ctypes.data_as(C.POINTER(C.c_double)), w.ctypes.data_as(C.POINTER(C.c_double))) < 0:
        raise ValueError(order)
    return t, w


def halo_for(buffer_len, k_update=4096):
    lib = _lib.load()
    l, r = C.c_int64(), C.c_int64()
    check(lib.kk_rx_halo_for(int(buffer_len), int(k_update), C.byref(l), C.byref(r)), "kk_rx_halo_for")
    return l.value, r.value
