"""Seeded synthetic input generator for the KK receiver (transmitter + channel + ADC).

This module produces INPUTS only (raw 12-bit ADC codes, the DC offset d, the
symbol pattern, the constellation file contents).  It contains none of the
receiver's arithmetic (no sqrt/log front end, Hilbert transform, reconstruction,
equaliser or decision); it is shared by the oracle tests, the GPU tests and
bench.py as a data source only (task rule: "only the seeded input generators
serve both").

Workload shape follows PAPER.md Sec. 3 (l.64-70) and SURVEY.md 8(d):
  * 2^20-symbol PCG64 pattern, repeated once per 2^22-sample buffer
  * 1 GBaud, 1 % roll-off RRC, synthesised periodically by FFT at
    4 samples/symbol (the 4 GS/s ADC rate)
  * digitally inserted tone at 0.516 GHz = bin 541065 of the 2^22 grid
    (11 MHz gap above the 0.505 GHz band edge)
  * CSPR = tone power / signal power (OSNR power includes the tone)
  * ASE noise loading at a given OSNR (0.1 nm = 12.5 GHz reference):
      one_sided  -- complex AWGN confined to the signal band (field stays
                    single-sideband; closed-form BER applies)
      two_sided  -- physical: flat over the 5 GHz optical BPF,
                    synthesised at 8 GS/s, square-law detected, ideal 2 GHz
                    anti-alias filter, decimated to 4 GS/s
  * ideal photodiode, 12-bit AC-coupled ADC: the pool mean is
    removed, gain g fills +-2047 for the noiseless swing (with an analytic noise
    headroom), codes are rint + clip to [-2048, 2047] int16
  * side output d = float32(g * mean(I)) -- the DC term the receiver adds back
    (static, optimised offline; here given exactly)

Noise is drawn per buffer from SeedSequence(seed_noise).spawn(n_pool); each
buffer's filtering is circular over that buffer (every buffer holds an integer
number of signal and tone periods, so the noiseless part is exactly periodic).
Streams are the pool cycled in order, so any halo is well defined.
"""
from __future__ import annotations

import hashlib
import os
from dataclasses import dataclass, asdict

import numpy as np
import scipy.fft as sfft

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CONST_DIR = os.path.join(ROOT, "data", "constellations")

BAUD = 1e9
FS = 4e9
ROLLOFF = 0.01
TONE_HZ = 0.516e9
REF_BW = 12.5e9       # 0.1 nm at 1550 nm
BPF_HALF = 2.5e9      # 5 GHz optical BPF
ADC_AA = 2.0e9        # ideal anti-alias at fs/2


def load_constellation(name: str):
    """Read data/constellations/<name>.txt ('<re> <im> <bits>' per line)."""
    return load_constellation_file(os.path.join(CONST_DIR, name + ".txt"))


def load_constellation_file(path: str):
    """Read a SPEC.md l.89 constellation file ('<re> <im> <label bits>' per line, '#'
    comments); points scaled to unit mean power, labels parsed as binary strings."""
    pts, labs = [], []
    with open(path) as f:
        for line in f:
            line = line.split("#", 1)[0].strip()
            if line:
                r, i, b = line.split()
                pts.append(complex(float(r), float(i)))
                labs.append(int(b, 2))
    p = np.array(pts, dtype=np.complex128)
    p = p / np.sqrt(np.mean(np.abs(p) ** 2))
    return p, np.array(labs, dtype=np.int64)


@dataclass(frozen=True)
class LinkConfig:
    fmt: str
    cspr_db: float
    osnr_db: float | None = None     # None = noiseless (back-to-back)
    noise: str = "one_sided"         # "one_sided" | "two_sided"
    buffer_len: int = 1 << 22
    pattern_len: int | None = None   # symbols; default buffer_len // 4
    tone_bin: int | None = None      # default round(0.516 GHz / 4 GS/s * N)
    seed_pat: int = 1
    seed_noise: int = 1000
    adc_bits: int = 12
    adc_bw_hz: float | None = None   # PD + ADC bandwidth (Gaussian, 3 dB at adc_bw_hz); None = ideal

    @property
    def n_sym(self):
        return self.buffer_len // 4

    @property
    def p_len(self):
        return self.pattern_len or self.n_sym

    @property
    def tbin(self):
        if self.tone_bin is not None:
            return int(self.tone_bin)
        return int(round(TONE_HZ / FS * self.buffer_len))

    def key(self):
        return hashlib.sha1(repr(sorted(asdict(self).items())).encode()).hexdigest()[:16]


@dataclass
class Pool:
    cfg: LinkConfig
    codes: np.ndarray        # int16 [n_pool, N]
    dc_offset: np.float32    # d = g * mean(I)
    gain: float
    pattern: np.ndarray      # uint8 [P] symbol indices
    points: np.ndarray
    labels: np.ndarray
    noise_var: float         # complex field noise variance per 4 GS/s sample (in-band)

    @property
    def n_pool(self):
        return self.codes.shape[0]


def rrc_response(f_baud, beta):
    """Root-raised-cosine amplitude response, f in units of the baud rate."""
    f = np.abs(f_baud)
    h = np.zeros_like(f)
    f1 = (1 - beta) / 2
    f2 = (1 + beta) / 2
    h[f <= f1] = 1.0
    m = (f > f1) & (f <= f2)
    h[m] = np.sqrt(0.5 * (1 + np.cos(np.pi / beta * (f[m] - f1))))
    return h


def make_pattern(m, p_len, seed):
    """'The 2^20 N-ary symbol sequence is generated using PCG64'."""
    return np.random.Generator(np.random.PCG64(seed)).integers(0, m, p_len).astype(np.uint8)


def signal_period(points, pattern):
    """Periodic 1 %-RRC shaping at 4 sps by FFT over one pattern period; unit power."""
    p_len = len(pattern)
    up = np.zeros(4 * p_len, dtype=np.complex128)
    up[::4] = points[pattern.astype(np.int64)]
    f = sfft.fftfreq(4 * p_len, d=0.25)  # in units of the baud rate
    s = sfft.ifft(sfft.fft(up, workers=-1) * rrc_response(f, ROLLOFF), workers=-1)
    return s / np.sqrt(np.mean(np.abs(s) ** 2))


def _tone(cfg, c):
    n = np.arange(cfg.buffer_len, dtype=np.int64)
    ph = np.mod(np.int64(cfg.tbin) * n, np.int64(cfg.buffer_len)).astype(np.float64)
    return np.sqrt(c) * np.exp(2j * np.pi * ph / cfg.buffer_len)


def clean_field(cfg, points, pattern):
    """s + tone for one buffer (buffer-local tone phase)."""
    s = signal_period(points, pattern)
    reps = cfg.buffer_len // len(s)
    assert reps * len(s) == cfg.buffer_len, "buffer must hold whole pattern periods"
    c = 10 ** (cfg.cspr_db / 10)
    return np.tile(s, reps) + _tone(cfg, c)


def noise_psd(cfg):
    """N0 (per Hz) such that N0 * 12.5 GHz = P_total 10^(-OSNR/10), P_total = 1 + c."""
    c = 10 ** (cfg.cspr_db / 10)
    return (1 + c) * 10 ** (-cfg.osnr_db / 10) / REF_BW


def _noise_intensity(cfg, e_clean, rng):
    """Intensity |E + n|^2 at 4 GS/s for one buffer (noise mode of cfg)."""
    n_buf = cfg.buffer_len
    n0 = noise_psd(cfg)
    if cfg.noise == "one_sided":
        sig = np.sqrt(n0 * FS / 2)
        w = rng.standard_normal(n_buf) + 1j * rng.standard_normal(n_buf)
        w *= sig
        f = sfft.fftfreq(n_buf, d=1 / FS)
        keep = np.abs(f) <= (1 + ROLLOFF) / 2 * BAUD
        W = sfft.fft(w, workers=-1)
        W[~keep] = 0
        e = e_clean + sfft.ifft(W, workers=-1)
        return np.abs(e) ** 2
    if cfg.noise == "two_sided":
        n8 = 2 * n_buf
        F = sfft.fft(e_clean, workers=-1)
        F8 = np.zeros(n8, dtype=np.complex128)
        h = n_buf // 2
        F8[:h] = F[:h]
        F8[n8 - h:] = F[h:]
        e8 = sfft.ifft(F8, workers=-1) * 2.0
        sig = np.sqrt(n0 * 2 * FS / 2)
        w = rng.standard_normal(n8) + 1j * rng.standard_normal(n8)
        w *= sig
        f8 = sfft.fftfreq(n8, d=1 / (2 * FS))
        W = sfft.fft(w, workers=-1)
        W[np.abs(f8) > BPF_HALF] = 0
        e8 += sfft.ifft(W, workers=-1)
        i8 = np.abs(e8) ** 2
        I8 = sfft.fft(i8, workers=-1)
        sub = np.concatenate([I8[:h], I8[n8 - h:]])
        sub[h] = 0.0  # 2 GHz bin (ideal anti-alias, exclusive)
        # i8 band-limited to |f| < 2 GHz => i4[n] = i8[2n] = 0.5 * ifft_N(sub)[n]
        return 0.5 * sfft.ifft(sub, workers=-1).real
    raise ValueError(cfg.noise)


def adc_filter(intens, bw_hz):
    """Finite PD + ADC bandwidth on the detected intensity (the paper's 1 GHz ADC,
    PAPER l.68; error-floor mechanism l.70, l.167): Gaussian low-pass |H(f)| =
    exp(-(ln 2 / 2) (f / bw)^2) (3 dB at bw), circular over each buffer period."""
    x = np.atleast_2d(np.asarray(intens, dtype=np.float64))
    f = sfft.rfftfreq(x.shape[-1], d=1 / FS)
    hf = np.exp(-0.5 * np.log(2.0) * (f / bw_hz) ** 2)
    y = sfft.irfft(sfft.rfft(x, axis=-1, workers=-1) * hf, n=x.shape[-1], axis=-1, workers=-1)
    return y.reshape(np.shape(intens))


def adc_gain(cfg: LinkConfig, i_clean=None):
    """Deterministic ADC gain: the noiseless swing fills +-(2^(b-1)-1) times an
    analytic headroom of 4 sigma of the signal-ASE beat term (function of the
    config only, so a noiseless training buffer can use the same gain)."""
    if i_clean is None:
        pts, _ = load_constellation(cfg.fmt)
        i_clean = np.abs(clean_field(cfg, pts, make_pattern(len(pts), cfg.p_len, cfg.seed_pat))) ** 2
    peak0 = float(np.max(np.abs(i_clean - i_clean.mean())))
    c = 10 ** (cfg.cspr_db / 10)
    if cfg.osnr_db is None:
        nv, headroom = 0.0, 1.0
    else:
        band = (1 + ROLLOFF) * BAUD if cfg.noise == "one_sided" else 2 * BPF_HALF
        nv = noise_psd(cfg) * band
        headroom = 1.0 + 4.0 * np.sqrt(2.0 * (1 + c) * nv) / peak0
    full = 2 ** (cfg.adc_bits - 1) - 1
    return full / (headroom * peak0), nv


_GEN_CTX = None  # (cfg, e_clean) inherited by forked generator workers


def _noise_worker(seq):
    cfg, e_clean = _GEN_CTX
    return _noise_intensity(cfg, e_clean, np.random.Generator(np.random.PCG64(seq)))


def make_pool(cfg: LinkConfig, n_pool: int = 1, cache: bool = True, noiseless: bool = False) -> Pool:
    """Generate n_pool distinct buffers of raw ADC codes for cfg.

    noiseless=True gives the training buffer of the same config: identical
    signal and ADC gain, no ASE (used to fit the static EQ)."""
    cache_path = None
    if noiseless:
        n_pool = 1
    if cache:
        d = os.environ.get("KKRX_CACHE", "/tmp/kkrx_cache")
        cache_path = os.path.join(d, f"pool_{cfg.key()}_{n_pool}_{int(noiseless)}.npz")
        if os.path.exists(cache_path):
            try:
                z = np.load(cache_path)
                pts, labs = load_constellation(cfg.fmt)
                return Pool(cfg, z["codes"], np.float32(z["d"]), float(z["g"]), z["pattern"], pts, labs,
                            float(z["nv"]))
            except Exception:
                pass
    pts, labs = load_constellation(cfg.fmt)
    pattern = make_pattern(len(pts), cfg.p_len, cfg.seed_pat)
    e_clean = clean_field(cfg, pts, pattern)
    i_clean = np.abs(e_clean) ** 2
    gain, nv = adc_gain(cfg, i_clean)
    intens = np.empty((n_pool, cfg.buffer_len), dtype=np.float64)
    if cfg.osnr_db is None or noiseless:
        intens[:] = i_clean
    else:
        seqs = np.random.SeedSequence(cfg.seed_noise).spawn(n_pool)
        import multiprocessing as mp
        procs = min(n_pool, os.cpu_count() or 1, int(os.environ.get("KKRX_GEN_PROCS", "16")))
        if procs > 1 and n_pool >= 4 and cfg.buffer_len >= (1 << 20) and not mp.current_process().daemon:
            # buffers in parallel processes (same per-buffer seeds and arithmetic: identical codes)
            global _GEN_CTX
            _GEN_CTX = (cfg, e_clean)
            with mp.get_context("fork").Pool(procs) as workers:
                for b, row in enumerate(workers.imap(_noise_worker, seqs)):
                    intens[b] = row
            _GEN_CTX = None
        else:
            for b in range(n_pool):
                intens[b] = _noise_intensity(cfg, e_clean, np.random.Generator(np.random.PCG64(seqs[b])))
    if cfg.adc_bw_hz is not None:
        intens = adc_filter(intens, cfg.adc_bw_hz)
    full = 2 ** (cfg.adc_bits - 1) - 1
    mean_i = float(intens.mean())
    codes = np.clip(np.rint(gain * (intens - mean_i)), -(full + 1), full).astype(np.int16)
    d = np.float32(gain * mean_i)
    pool = Pool(cfg, codes, d, gain, pattern, pts, labs, nv)
    if cache_path is not None:
        try:
            os.makedirs(os.path.dirname(cache_path), exist_ok=True)
            tmp = cache_path + f".tmp{os.getpid()}.npz"
            np.savez(tmp, codes=codes, d=d, g=gain, pattern=pattern, nv=nv)
            os.replace(tmp, cache_path)
        except OSError:
            pass
    return pool


def pack12(codes: np.ndarray) -> np.ndarray:
    """int16 ADC codes (12-bit range) -> the packed 12-bit byte format of a 12-bit ADC:
    two two's-complement codes per 3 bytes, little-endian (b0 = c0[7:0],
    b1 = c0[11:8] | c1[3:0] << 4, b2 = c1[11:4]).  Input format only (no method arithmetic)."""
    c = np.asarray(codes, dtype=np.int16)
    assert c.size % 2 == 0
    u = (c.astype(np.int32) & 0xFFF).reshape(-1, 2)
    out = np.empty((u.shape[0], 3), dtype=np.uint8)
    out[:, 0] = u[:, 0] & 0xFF
    out[:, 1] = ((u[:, 0] >> 8) & 0x0F) | ((u[:, 1] & 0x0F) << 4)
    out[:, 2] = (u[:, 1] >> 4) & 0xFF
    return out.reshape(-1)


def make_stream(pool: Pool, n_buffers: int, left: int, right: int, first: int = 0):
    """Contiguous int16 stream holding stream buffers first .. first+n_buffers-1
    plus `left` samples before and `right` after, cycling the pool in order.
    Returns (stream, offset_of_buffer_first)."""
    n_buf = pool.cfg.buffer_len
    flat = pool.codes.reshape(-1)
    total = flat.size
    start = first * n_buf - left
    idx = (np.arange(start, start + left + n_buffers * n_buf + right, dtype=np.int64)) % total
    return flat[idx], left
