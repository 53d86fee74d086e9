"""Plain float64 CPU oracle of the KK receiver hot path.

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import, call or execute anything under
oracle/.  The product path (paper_2108_07004_b200/) never imports it and shares
no code, tables or constants with it.

Every function follows one step of the chain described in PAPER.md Sec. 2
(l.45-53, "Digital signal processing chain"), in the paper's order:

  S1 front end        PAPER l.47 "converting samples received as 12-bit fixed point
                      to 32-bit floating point numbers, adding the appropriate DC
                      offset, and performing the square root and logarithm"
  S2 Hilbert          PAPER l.47 "enabled by a pair of 100% overlap-save 1024-point
                      FFTs, the phase of the optical signal is recovered by a
                      frequency-domain Hilbert transform"
  S3 reconstruct      PAPER l.47 "This phase is combined with the amplitude
                      calculated in step 1 to reconstruct the optical signal which
                      is subsequently downconverted"
  S4 static EQ + 4->2 PAPER l.47 "Another pair of FFTs supports frequency-domain
                      static equalization and resampling from 4 to 2
                      samples-per-symbol"; l.53 "203-tap static frequency-domain
                      equalizer"
  S5 WL DD-LMS        PAPER l.47 "a 4-tap adaptive time-domain widely-linear DDLMS
                      equalizer"; l.53 "after initial setup and convergence using a
                      training sequence, it is updated in a blind decision-directed
                      fashion where part of a buffer is used to update equalizer
                      taps for subsequent buffers"
  S6 decision         PAPER l.47/l.53 "minimum Euclidean distance"
  S7 demap + count    PAPER l.47 "demapped into bits"; l.68 "Error counting"

Where the paper is silent the readings R1..R17 of DESIGN.md (= SURVEY.md 8(c)
items 1-17) are followed; each function names the readings it uses.

Parity unpinned: wl_lms_update's exact tap *trajectory* -- the paper
fixes neither mu nor the update schedule K, so only properties are pinned (Lipschitz
bound, ablation, convergence to the Wiener gain SNR/(1+SNR)); the GPU parity tests
compare the trajectory element by element against this function, not against a paper
value.

Precision: float64 throughout (numpy), integer phase arithmetic for the tone.
Library primitives used as single steps: numpy.fft.fft / ifft (S2, one call per
1024-point block, exactly as the method states it).  No blocking, fusion or
reordering beyond the definitions below.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

# 1024-point FFTs; reading R2: hop 512, keep the centre 512.
HILBERT_NFFT = 1024
HILBERT_HOP = 512
HILBERT_DISCARD = 256
# 203-tap static equaliser; reading R4: centred FIR, taps -101..101.
FIR_TAPS = 203
FIR_HALF = 101
# 4 -> 2 samples per symbol; 4 taps in the adaptive equaliser.
SPS = 4
WL_TAPS = 4

UPD_DD_SOFT, UPD_PILOT, UPD_DD_HARD = 0, 1, 2


# ----------------------------------------------------------------------------
# O1 / S1 front end
# ----------------------------------------------------------------------------
def pre_equalize(codes, d, g):
    """Pre-KK static equaliser (PAPER l.167 [chenKKFE]): a short real
    FIR on the detected intensity before sqrt/log, undoing the PD/ADC roll-off,
        v'[n] = sum_{k=-h..h} g_k (code[n - k] + d),   g_k = g[k + h],  len(g) = 2h + 1.
    Plain direct convolution; returns v' for n = h .. len(codes)-1-h (length len - 2h)."""
    v = np.asarray(codes, dtype=np.float64) + np.float64(d)
    g = np.asarray(g, dtype=np.float64)
    h = (len(g) - 1) // 2
    assert len(g) == 2 * h + 1
    n = len(v) - 2 * h
    out = np.zeros(n, dtype=np.float64)
    for k in range(-h, h + 1):
        out += g[k + h] * v[h - k: h - k + n]
    return out


def frontend_v(v, v_min=1.0):
    """S1 on intensities already holding the DC offset: clamp, sqrt, log."""
    v = np.asarray(v, dtype=np.float64)
    clipped = v < v_min
    v = np.maximum(v, np.float64(v_min))
    return np.sqrt(v), 0.5 * np.log(v), clipped


def frontend(codes, d, v_min=1.0):
    """v = max(code + d, v_min); a = sqrt(v); l = ln a = 0.5 ln v.

    PAPER l.47 (fixed->float, DC offset, sqrt, log) and l.51 (the DC term lost
    by the AC-coupled ADC is added back).  Reading R9: v < v_min is clamped and
    counted instead of raising (SPEC.md l.344 raises).
    Returns (a, l, clipped_mask)."""
    v = np.asarray(codes, dtype=np.float64) + np.float64(d)
    clipped = v < v_min
    v = np.maximum(v, np.float64(v_min))
    a = np.sqrt(v)
    l = 0.5 * np.log(v)
    return a, l, clipped


# ----------------------------------------------------------------------------
# O2 / S2 Hilbert (the method is blockwise, not the ideal Hilbert transform)
# ----------------------------------------------------------------------------
def hilbert_mask(nfft=HILBERT_NFFT):
    """Frequency response of phi = -H{l}: +i*sgn(k), sgn(0)=sgn(N/2)=0.

    Reading R1: the signal sits below the tone (edge 0.505 GHz,
    tone 0.516 GHz), so in the tone frame the field is A + s' with s' at
    negative frequencies only; ln|E| and arg E then form the Hilbert pair
    phi = -H{ln a} with H <-> -i*sgn(k).  DC and Nyquist bins are zeroed
    (SPEC.md l.352)."""
    k = np.arange(nfft)
    m = np.zeros(nfft, dtype=np.complex128)
    m[(k > 0) & (k < nfft // 2)] = 1j
    m[k > nfft // 2] = -1j
    return m


def hilbert_phase(l, pos0, j_first, j_last):
    """Blockwise phase phi for the 512-sample chunks j = j_first..j_last.

    Chunk j covers stream positions [512 j, 512 j + 512) and is taken from the
    centre of the 1024-point window [512 j - 256, 512 j + 768)  (PAPER l.47
    "100% overlap-save 1024-point FFTs"; reading R2).  Per window: FFT,
    multiply by hilbert_mask(), inverse FFT, real part, keep the centre.
    `l[i]` is the log-amplitude at position pos0 + i.
    Returns phi for positions [512 j_first, 512 (j_last + 1))."""
    mask = hilbert_mask()
    n_chunks = j_last - j_first + 1
    out = np.empty(n_chunks * HILBERT_HOP, dtype=np.float64)
    for c in range(n_chunks):
        j = j_first + c
        start = HILBERT_HOP * j - HILBERT_DISCARD - pos0
        if start < 0 or start + HILBERT_NFFT > len(l):
            raise ValueError("log-amplitude window does not cover Hilbert block %d" % j)
        w = l[start:start + HILBERT_NFFT]
        phi_w = np.fft.ifft(np.fft.fft(w) * mask).real
        out[c * HILBERT_HOP:(c + 1) * HILBERT_HOP] = phi_w[HILBERT_DISCARD:HILBERT_DISCARD + HILBERT_HOP]
    return out


# ----------------------------------------------------------------------------
# O3 / S3 reconstruction, carrier removal, downconversion
# ----------------------------------------------------------------------------
def carrier_amplitude(d, cspr_db):
    """A_hat = sqrt(d * c / (1 + c)), c = 10^(CSPR/10)  (reading R6).

    d = g * mean(I) and mean(I) = P_s (1 + c) for unit-power signal plus tone of
    power c * P_s (total power includes the tone), so
    d c / (1 + c) = g * A^2."""
    c = 10.0 ** (np.float64(cspr_db) / 10.0)
    return np.sqrt(np.float64(d) * c / (1.0 + c))


def tone_phase(positions, tone_bin, buffer_len):
    """theta_n = 2 pi ((tone_bin * n) mod N) / N with exact integer reduction.

    Reading R7: tone_bin = 541065 for N = 2^22 (0.516 GHz at 4 GS/s),
    so every buffer holds an integer number of tone periods and theta is
    buffer-local.  Python integers: no overflow."""
    n = np.asarray(positions, dtype=object)
    p = np.array([(int(tone_bin) * int(x)) % int(buffer_len) for x in n], dtype=np.float64)
    return 2.0 * np.pi * p / float(buffer_len)


def tone_phase_fast(positions, tone_bin, buffer_len):
    """Same as tone_phase() using int64 when |tone_bin * n| < 2^63 (checked)."""
    pos = np.asarray(positions, dtype=np.int64)
    if pos.size and (abs(int(tone_bin)) * int(np.max(np.abs(pos)) + 1) >= 2 ** 62):
        return tone_phase(positions, tone_bin, buffer_len)
    p = np.mod(np.int64(tone_bin) * pos, np.int64(buffer_len)).astype(np.float64)
    return 2.0 * np.pi * p / float(buffer_len)


def reconstruct_downconvert(a, phi, a_hat, theta):
    """E_s[n] = (a[n] e^{i phi[n]} - A_hat) e^{+i theta_n}.

    PAPER l.47 "combined with the amplitude ... to reconstruct the optical
    signal which is subsequently downconverted".  Readings R1 (sign e^{+i theta}
    because the signal is below the tone) and R6 (static carrier removal)."""
    return (a * np.exp(1j * phi) - a_hat) * np.exp(1j * theta)


# ----------------------------------------------------------------------------
# O4 / S4 static equaliser and 4 -> 2 resampling (exact LTI: plain definition)
# ----------------------------------------------------------------------------
def static_eq_resample(e_s, pos0, h, x2_first, x2_count):
    """x2[m] = sum_{i=-101}^{101} h_i * E_s[2m - i]   (direct form).

    PAPER l.47/l.53; readings R3, R4, R5: a centred 203-tap complex FIR at
    4 sps followed by exact decimation by 2 (the frequency-domain method with a
    spectral fold computes exactly this, independent of FFT size).
    `e_s[i]` is E_s at position pos0 + i; `h[t]` is tap i = t - 101.
    Returns x2[m] for m in [x2_first, x2_first + x2_count)."""
    h = np.asarray(h, dtype=np.complex128)
    assert len(h) == FIR_TAPS
    m = np.arange(x2_first, x2_first + x2_count, dtype=np.int64)
    out = np.zeros(x2_count, dtype=np.complex128)
    for t in range(FIR_TAPS):
        i = t - FIR_HALF
        idx = 2 * m - i - pos0
        if idx[0] < 0 or idx[-1] >= len(e_s):
            raise ValueError("E_s does not cover the FIR reach")
        out += h[t] * e_s[idx]
    return out


# ----------------------------------------------------------------------------
# O5 / S5 widely-linear LMS update pass
# ----------------------------------------------------------------------------
def wl_regressor(x2_at, n):
    """u_n = (x2[2n+1], x2[2n], x2[2n-1], x2[2n-2])  (reading R10: T/2-spaced
    taps, centre tap index 1 on x2[2n])."""
    return np.array([x2_at(2 * n + 1), x2_at(2 * n), x2_at(2 * n - 1), x2_at(2 * n - 2)])


def wl_output(w, g, u):
    """y = w^T u + g^T u*  (SPEC.md l.388 convention, no conjugate on w)."""
    return np.sum(w * u) + np.sum(g * np.conj(u))


def decide_two(y, points):
    """Brute force D_k = |y - p_k|^2; k1 = argmin (lowest index on ties);
    D(2) = second-smallest value over k != k1."""
    d = (y.real - points.real) ** 2 + (y.imag - points.imag) ** 2
    k1 = int(np.argmin(d))
    d1 = d[k1]
    d2 = np.min(np.delete(d, k1))
    return k1, d1, d2


def wl_lms_update(x2_at, n_start, k_steps, w_init, g_init, mu, points, tau, mode,
                  pattern=None, ref_offset=0):
    """Run the LMS update over symbols n_start .. n_start + k_steps - 1 in order.

    PAPER l.53: "part of a buffer is used to update equalizer taps for
    subsequent buffers"; blind decision-directed after training.  Reading R10:
    per step
        y  = w.u + g.u*;  D_k = |y - p_k|^2;  k1 = argmin;  D(2) second smallest
        ref = p_k1 (DD) or p_pattern[(n + n_off) mod P] (PILOT)
        gamma = 1 (PILOT or tau == 0) else min(1, (D(2) - D(1)) / tau)
        e = gamma (ref - y);  w += mu e u*;  g += mu e u
    Returns (w, g, gated_steps, mean |e|^2)."""
    w = np.array(w_init, dtype=np.complex128).copy()
    g = np.array(g_init, dtype=np.complex128).copy()
    gated = 0
    esum = 0.0
    for s in range(k_steps):
        n = n_start + s
        u = wl_regressor(x2_at, n)
        y = wl_output(w, g, u)
        k1, d1, d2 = decide_two(y, points)
        if mode == UPD_PILOT:
            ref = points[int(pattern[(n + ref_offset) % len(pattern)])]
            gamma = 1.0
        else:
            ref = points[k1]
            if tau == 0.0 or mode == UPD_DD_HARD:
                gamma = 1.0
            else:
                gamma = min(1.0, (d2 - d1) / tau)
        if gamma < 1.0:
            gated += 1
        e = gamma * (ref - y)
        esum += abs(e) ** 2
        w = w + mu * e * np.conj(u)
        g = g + mu * e * u
    return w, g, gated, esum / max(k_steps, 1)


# ----------------------------------------------------------------------------
# O6 / S5' + S6 apply and decide
# ----------------------------------------------------------------------------
def wl_apply(x2, x2_first, n_first, n_count, w, g):
    """y_n = w.u_n + g.u_n* for n in [n_first, n_first + n_count), fixed taps.
    `x2[i]` is x2 index x2_first + i."""
    n = np.arange(n_first, n_first + n_count, dtype=np.int64)
    u = [x2[2 * n + 1 - x2_first], x2[2 * n - x2_first], x2[2 * n - 1 - x2_first], x2[2 * n - 2 - x2_first]]
    y = np.zeros(n_count, dtype=np.complex128)
    for k in range(WL_TAPS):
        y += w[k] * u[k] + g[k] * np.conj(u[k])
    return y


def decide(y, points, chunk=1 << 15):
    """d_n = argmin_k |y_n - p_k|^2 (lowest index on ties) by brute force, and
    the exact distance of y_n to the boundary of its Voronoi cell
        m_n = min_{k != d} (D_k - D_d) / (2 |p_k - p_d|)
    (used only to define the parity exempt set)."""
    y = np.asarray(y, dtype=np.complex128)
    dec = np.empty(len(y), dtype=np.int64)
    margin = np.empty(len(y), dtype=np.float64)
    pd = np.abs(points[:, None] - points[None, :])
    for s in range(0, len(y), chunk):
        yy = y[s:s + chunk]
        dk = (yy.real[:, None] - points.real[None, :]) ** 2 + (yy.imag[:, None] - points.imag[None, :]) ** 2
        dd = np.argmin(dk, axis=1)
        dmin = dk[np.arange(len(yy)), dd]
        sep = pd[dd]  # |p_k - p_d|
        with np.errstate(divide="ignore", invalid="ignore"):
            mm = (dk - dmin[:, None]) / (2.0 * sep)
        mm[np.arange(len(yy)), dd] = np.inf
        dec[s:s + chunk] = dd
        margin[s:s + chunk] = mm.min(axis=1)
    return dec, margin


# ----------------------------------------------------------------------------
# O7 / S7 demap + count
# ----------------------------------------------------------------------------
def popcount(x):
    x = np.asarray(x, dtype=np.int64)
    c = np.zeros_like(x)
    for b in range(8):
        c += (x >> b) & 1
    return c


def count_errors(dec, ref_idx, labels):
    """sym_err = #(d != ref), bit_err = sum popcount(lab[d] xor lab[ref])
    (PAPER l.68 error counting)."""
    dec = np.asarray(dec, dtype=np.int64)
    ref_idx = np.asarray(ref_idx, dtype=np.int64)
    labels = np.asarray(labels, dtype=np.int64)
    bits_per = int(np.log2(len(labels)))
    return dict(
        sym_errors=int(np.sum(dec != ref_idx)),
        bit_errors=int(np.sum(popcount(labels[dec] ^ labels[ref_idx]))),
        symbols=int(len(dec)),
        bits=int(len(dec) * bits_per),
    )


# ----------------------------------------------------------------------------
# Composition (one buffer), = kk_rx_process on the same int16 window
# ----------------------------------------------------------------------------
@dataclass
class RxParams:
    buffer_len: int
    cspr_db: float
    dc_offset: float            # float32 value used bit-for-bit by both sides
    fir: np.ndarray             # complex [203], tap i = t - 101
    points: np.ndarray          # complex [M]
    labels: np.ndarray          # int [M]
    tone_bin: int = 541065
    w_init: np.ndarray = field(default_factory=lambda: np.array([0, 1, 0, 0], dtype=np.complex128))
    g_init: np.ndarray = field(default_factory=lambda: np.zeros(4, dtype=np.complex128))
    mu: float = 1e-3
    k_update: int = 4096
    sub_block: int | None = None   # L symbols; None = whole buffer
    gate_tau: float = -1.0         # <0: d_min^2/4
    update_mode: int = UPD_DD_SOFT
    v_min: float = 1.0
    pattern: np.ndarray | None = None   # ref indices (error-count reference)
    ref_offset: int = 0
    pre_fir: np.ndarray | None = None   # real [2h+1], pre-KK intensity equaliser (NEXT-3), h <= 8


def d_min(points):
    d = np.abs(points[:, None] - points[None, :])
    d[np.arange(len(points)), np.arange(len(points))] = np.inf
    return float(d.min())


def required_left(k_update):
    """Raw samples needed before the buffer: the update segment reaches x2
    position -(4K+4); the FIR reaches 101 more; Hilbert chunks are on the
    512 grid with a 256 window margin."""
    need = 4 * k_update + 4 + FIR_HALF
    return HILBERT_HOP * (-(-need // HILBERT_HOP)) + HILBERT_DISCARD


def required_right():
    """x2 up to position N-2 needs E_s up to N+99 -> Hilbert chunk N/512 whose
    window reaches N + 768."""
    return HILBERT_HOP + HILBERT_DISCARD


def receive(window, left, p: RxParams, want_stages=False):
    """Process one buffer: `window[i]` is the raw code at buffer position i - left.

    Steps S1..S7 in the paper's order.  The update pass for sub-block q runs
    over symbols qL-K .. qL-1 from W_init (reading R10: restart per sub-block
    so buffers are independent), then the fixed taps are applied to
    [qL, qL+L)."""
    n_buf = int(p.buffer_len)
    n_sym = n_buf // SPS
    L = n_sym if p.sub_block is None else int(p.sub_block)
    assert n_sym % L == 0
    K = int(p.k_update)
    window = np.asarray(window)
    right = len(window) - left - n_buf
    hp = 0 if p.pre_fir is None else (len(p.pre_fir) - 1) // 2
    if left < required_left(K) + hp or right < required_right() + hp:
        raise ValueError("window too small: need left>=%d right>=%d" % (required_left(K) + hp, required_right() + hp))
    pos0 = -left
    # S1 (with the optional pre-KK intensity equaliser: the window loses h samples per side)
    if p.pre_fir is not None:
        h = (len(p.pre_fir) - 1) // 2
        a, l, clipped = frontend_v(pre_equalize(window, p.dc_offset, p.pre_fir), p.v_min)
        window = window[h:len(window) - h]
        left -= h
        pos0 = -left
    else:
        a, l, clipped = frontend(window, p.dc_offset, p.v_min)
    # S2 on every whole chunk the window supports
    j_first = -(-(pos0 + HILBERT_DISCARD) // HILBERT_HOP)
    j_last = (pos0 + len(window) - (HILBERT_NFFT - HILBERT_DISCARD)) // HILBERT_HOP
    phi = hilbert_phase(l, pos0, j_first, j_last)
    e_pos0 = HILBERT_HOP * j_first
    pos = np.arange(e_pos0, e_pos0 + len(phi), dtype=np.int64)
    # S3
    a_hat = carrier_amplitude(p.dc_offset, p.cspr_db)
    theta = tone_phase_fast(pos, p.tone_bin, n_buf)
    e_s = reconstruct_downconvert(a[pos - pos0], phi, a_hat, theta)
    # S4 over the x2 range the update pass and the apply need
    x2_first = 2 * (-K) - 2
    x2_last = 2 * (n_sym - 1) + 1
    x2 = static_eq_resample(e_s, e_pos0, p.fir, x2_first, x2_last - x2_first + 1)

    def x2_at(m):
        return x2[m - x2_first]

    tau = p.gate_tau
    if tau < 0:
        tau = d_min(p.points) ** 2 / 4.0
    # S5 update + S5' apply + S6 decide, per sub-block
    taps = []
    y = np.empty(n_sym, dtype=np.complex128)
    gated = 0
    emean = []
    for q in range(n_sym // L):
        w, g, gq, em = wl_lms_update(x2_at, q * L - K, K, p.w_init, p.g_init, p.mu, p.points, tau,
                                     p.update_mode, p.pattern, p.ref_offset)
        gated += gq
        emean.append(em)
        taps.append((w, g))
        y[q * L:(q + 1) * L] = wl_apply(x2, x2_first, q * L, L, w, g)
    dec, margin = decide(y, p.points)
    out = dict(decisions=dec, labels_out=np.asarray(p.labels)[dec], margin=margin, taps=taps,
               gated_updates=gated, clipped=int(np.sum(clipped[left:left + n_buf])), y=y,
               e_mean=np.array(emean))
    if p.pattern is not None:
        ref = np.asarray(p.pattern, dtype=np.int64)[(np.arange(n_sym) + p.ref_offset) % len(p.pattern)]
        out["ref"] = ref
        out.update(count_errors(dec, ref, p.labels))
    if want_stages:
        out.update(e_s=e_s, e_pos0=e_pos0, x2=x2, x2_first=x2_first, phi=phi, a_hat=a_hat)
    return out
