"""Init-time training (TOOL): LS fit of the 203-tap static equaliser and PILOT
convergence of the adaptive taps, on a known training sequence.

TEST / TOOL INFRASTRUCTURE ONLY (see oracle/kk_oracle.py header).

PAPER l.53: "the 203-tap static frequency-domain equalizer is optimized offline
using a training sequence every time that the data acquisition is initialized"
and "after initial setup and convergence using a training sequence" (adaptive).
Reading R4: the 203 taps are a centred complex FIR at 4 sps (tap i = -101..101)
fitted by least squares so that x2 at the symbol instants (4-sps position 4n,
reading R15) approximates the transmitted symbols.  The result is an INPUT of
kk_rx_create (param `fir`) and is committed under data/fir/ by
tools/make_fixtures.py, which calls only oracle/ (and synth/ for the input).
"""
from __future__ import annotations

import numpy as np

from . import kk_oracle as O


def field_after_s3(window, left, p: O.RxParams):
    """E_s for every whole Hilbert chunk of the window (oracle S1-S3)."""
    pos0 = -left
    a, l, _ = O.frontend(window, p.dc_offset, p.v_min)
    j_first = -(-(pos0 + O.HILBERT_DISCARD) // O.HILBERT_HOP)
    j_last = (pos0 + len(window) - (O.HILBERT_NFFT - O.HILBERT_DISCARD)) // O.HILBERT_HOP
    phi = O.hilbert_phase(l, pos0, j_first, j_last)
    e_pos0 = O.HILBERT_HOP * j_first
    pos = np.arange(e_pos0, e_pos0 + len(phi), dtype=np.int64)
    theta = O.tone_phase_fast(pos, p.tone_bin, p.buffer_len)
    e_s = O.reconstruct_downconvert(a[pos - pos0], phi, O.carrier_amplitude(p.dc_offset, p.cspr_db), theta)
    return e_s, e_pos0


def train_fir(window, left, p: O.RxParams, symbols_tx, n_first, n_count, ridge=1e-9, unbiased=False):
    """min_h sum_n |sum_t h[t] E_s[4n + 101 - t] - s_n|^2 + ridge ||h||^2.

    On a noisy training buffer (the live link of PAPER l.53) this least-squares fit is
    the sample MMSE filter: it also weighs the noise the KK front end folds into the
    band, so it constrains the stopband a noiseless fit leaves free.  The MMSE
    estimate is biased toward zero, x = g s + noise with g = <x, s>/<s, s> < 1, which
    shrinks the constellation against the fixed decision regions (S6); unbiased=True
    returns h / g (the unbiased MMSE filter, same SNR, unit gain on the training
    symbols).  DESIGN.md reading R4."""
    e_s, e_pos0 = field_after_s3(window, left, p)
    n = np.arange(n_first, n_first + n_count, dtype=np.int64)
    t = np.arange(O.FIR_TAPS, dtype=np.int64)
    idx = 4 * n[:, None] + O.FIR_HALF - t[None, :] - e_pos0
    A = e_s[idx]
    b = np.asarray(symbols_tx, dtype=np.complex128)
    AhA = A.conj().T @ A
    AhA += ridge * np.trace(AhA).real / O.FIR_TAPS * np.eye(O.FIR_TAPS)
    h = np.linalg.solve(AhA, A.conj().T @ b)
    if unbiased:
        x = A @ h
        g = np.vdot(b, x) / np.vdot(b, b)
        h = h / g
    return h


def train_prefir(window, target, d, h, ridge=1e-9):
    """Pre-KK intensity equaliser: real taps g[0..2h] minimising
    sum_n |sum_k g_k (window[n - k] + d) - (target[n] + d)|^2 (+ ridge) over the
    interior of the window; `target` = the same buffer's codes without the PD/ADC
    roll-off (the noiseless training pair of synth.generate)."""
    v = np.asarray(window, dtype=np.float64) + np.float64(d)
    t = np.asarray(target, dtype=np.float64) + np.float64(d)
    n = len(v) - 2 * h
    A = np.stack([v[h - k: h - k + n] for k in range(-h, h + 1)], axis=1)
    b = t[h: h + n]
    AtA = A.T @ A
    AtA += ridge * np.trace(AtA) / (2 * h + 1) * np.eye(2 * h + 1)
    return np.linalg.solve(AtA, A.T @ b)


def frame_sync_corr(e_s, e_pos0, points, pattern, n0, n_corr):
    """Frame synchronisation ("frame-sync correlation against the
    PCG64 pattern", the step before the FIR fit; the 2^20-symbol PCG64
    sequence is known to the receiver).  The received field at the symbol instants
    (4-sps position 4n, reading R15), y_n = E_s[4n], is correlated with the known pattern
    points over every cyclic lag k of the pattern:

        c(k) = sum_{n=0}^{n_corr-1} y_{n0+n} conj(p[(n0 + n + k) mod P]),  p = points[pattern]

    for all k at once, as a circular cross-correlation by FFT over the pattern period (a
    library primitive standing for the sum above; tests pin it against the direct sum)."""
    P = len(pattern)
    y = e_s[4 * (n0 + np.arange(n_corr, dtype=np.int64)) - e_pos0]
    q = np.conj(np.asarray(points)[np.asarray(pattern, dtype=np.int64)])
    ypad = np.zeros(P, dtype=np.complex128)
    ypad[:n_corr] = y
    # c'(m) = sum_j y_j q[(j + m) mod P] = IFFT(FFT(q) conj(FFT(conj(y))))(m), m = n0 + k
    cm = np.fft.ifft(np.fft.fft(q) * np.conj(np.fft.fft(np.conj(ypad))))
    return np.roll(cm, -n0)  # c[k] = c'(n0 + k)


def frame_sync(e_s, e_pos0, points, pattern, n0, n_corr):
    """The frame offset n_off = argmax_k |c(k)| (lowest k on ties): the symbol sent at
    buffer index n is pattern[(n + n_off) mod P].  Returns (n_off,
    c(n_off), mean over k of |c(k)|^2)."""
    c = frame_sync_corr(e_s, e_pos0, points, pattern, n0, n_corr)
    mag = np.abs(c) ** 2
    k = int(np.argmax(mag))
    return k, c[k], float(np.mean(mag))


def frame_sync_direct(e_s, e_pos0, points, pattern, n0, n_corr, k):
    """c(k) of frame_sync by the plain double sum (the definition), for pins."""
    P = len(pattern)
    n = np.arange(n_corr, dtype=np.int64)
    y = e_s[4 * (n0 + n) - e_pos0]
    p = np.asarray(points)[np.asarray(pattern, dtype=np.int64)[(n0 + n + k) % P]]
    return np.sum(y * np.conj(p))
