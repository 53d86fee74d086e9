"""Pins of the float64 oracle against things other than itself (-m "not gpu").

Each test names the paper passage / closed form / invariant it checks.  The
oracle is only trusted after these pass (task rule 3).  A plausible mistake
(wrong Hilbert sign, wrong downconversion sign, dropped 1/2 in the log, wrong
tap index, transposed operand) fails at least one of them.
"""
import json
import math
import os

import numpy as np
import pytest

from oracle import constellation as C
from oracle import kk_oracle as O
from oracle import metrics as Mx

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_numbers.json")))


# ---------------------------------------------------------------- S1 front end
def test_frontend_constant_code():
    """constant code c, offset d -> a = sqrt(c + d) everywhere;
    l = ln a (the factor 1/2 of ln v is pinned here)."""
    a, l, clip = O.frontend(np.full(100, 37, np.int16), np.float32(963.5))
    assert np.all(a == math.sqrt(1000.5))
    assert np.allclose(l, math.log(math.sqrt(1000.5)), rtol=0, atol=1e-15)
    assert not clip.any()


def test_frontend_clamp_and_count():
    """Reading R9: code + d < v_min is clamped to v_min and counted."""
    a, l, clip = O.frontend(np.array([-2048, 0, 5], np.int16), np.float32(10.0), v_min=1.0)
    assert clip.tolist() == [True, False, False]
    assert a[0] == 1.0 and l[0] == 0.0


# ---------------------------------------------------------------- S2 Hilbert
def _chunks_for(nsamp):
    """positions [0, nsamp) with whole Hilbert windows inside."""
    pos0 = 0
    j_first = 1
    j_last = (nsamp - 768) // 512
    return pos0, j_first, j_last


@pytest.mark.parametrize("k", [1, 7, 100, 255, 511])
def test_hilbert_bin_centred_tone(k):
    """H{cos} = sin exactly for a tone on the 1024-point grid (SPEC.md l.355,
    PAPER l.47).  phi = -H{l} (reading R1) so phi = -sin.  The reference
    argument is reduced with integers, so the only error is fp64 rounding."""
    n = np.arange(8192)
    psi = 0.3
    arg = 2 * np.pi * ((k * n) % 1024) / 1024 + psi
    l = np.cos(arg)
    pos0, jf, jl = _chunks_for(len(n))
    phi = O.hilbert_phase(l, pos0, jf, jl)
    ref = -np.sin(arg[512 * jf:512 * (jl + 1)])
    assert np.max(np.abs(phi - ref)) < 1e-12


def test_hilbert_constant_and_nyquist_zero():
    """Constant -> 0 (DC bin zeroed) and the Nyquist tone (-1)^n -> 0."""
    n = np.arange(4096)
    for l in (np.full(4096, 3.25), np.cos(np.pi * n)):
        phi = O.hilbert_phase(l, 0, 1, 5)
        assert np.max(np.abs(phi)) < 1e-12


def test_hilbert_direct_form_closed_kernel():
    """Direct circular convolution with the closed-form kernel of -i*sgn(k)
    (DC, Nyquist zeroed): h[q] = (2/1024) cot(pi q / 1024) for odd q, 0 for even
    q.  phi[512j + r] = -sum_m h[(256 + r - m) mod 1024] w_j[m]."""
    rng = np.random.default_rng(5)
    l = rng.standard_normal(4096)
    phi = O.hilbert_phase(l, 0, 1, 5)
    q = np.arange(1024)
    h = np.zeros(1024)
    odd = q % 2 == 1
    h[odd] = 2.0 / 1024 / np.tan(np.pi * q[odd] / 1024)
    for j in range(1, 6):
        w = l[512 * j - 256:512 * j + 768]
        for r in (0, 1, 255, 256, 511):
            val = -np.sum(h[(256 + r - np.arange(1024)) % 1024] * w)
            assert abs(val - phi[512 * (j - 1) + r]) < 1e-12


def test_hilbert_blockwise_is_periodically_time_varying():
    """The 1024/512 blockwise Hilbert is NOT the whole-buffer Hilbert (reported,
    not gated): a shift by 512 commutes, a shift by 256
    does not."""
    rng = np.random.default_rng(1)
    l = rng.standard_normal(8192)
    a = O.hilbert_phase(l, 0, 2, 10)
    b = O.hilbert_phase(np.roll(l, 512), 0, 3, 11)
    assert np.max(np.abs(a - b)) < 1e-12
    c = O.hilbert_phase(np.roll(l, 256), 0, 2, 10)
    assert np.max(np.abs(np.roll(a, 256)[512:-512] - c[512:-512])) > 1e-3


# ---------------------------------------------------------------- S3 reconstruction (exact MP field)
def _exact_mp_field(n, amp, tone_bin, nbuf, seed=3, ntones=40, depth=0.25):
    """E_tf = A exp(g), g a multitone on NEGATIVE bins of the 1024 grid, so
    ln|E_tf| and arg E_tf are an exact circular Hilbert pair in every window.
    Full field E = E_tf e^{+i theta} (tone above the signal).
    Returns (E, s_true) with s_true = E - A e^{i theta}."""
    rng = np.random.default_rng(seed)
    ks = rng.choice(np.arange(1, 400), ntones, replace=False)
    c = depth / ntones * (rng.standard_normal(ntones) + 1j * rng.standard_normal(ntones))
    g = np.zeros(len(n), dtype=np.complex128)
    for kk, cc in zip(ks, c):
        g += cc * np.exp(-2j * np.pi * ((kk * n) % 1024) / 1024)
    theta = 2 * np.pi * ((tone_bin * n) % nbuf) / nbuf
    e_tf = amp * np.exp(g)
    return e_tf * np.exp(1j * theta), (e_tf - amp) * np.exp(1j * theta)


def test_exact_minimum_phase_field_recovered():
    """KK exactness (PAPER l.47 S1-S3): for a strictly MP field
    whose log-spectrum lies on the 1024 grid the blockwise chain recovers the
    signal to fp64 rounding.  Also pins: the 1/2 in l = ln sqrt(v), the Hilbert
    sign (reading R1), the e^{+i theta} downconversion and A_hat."""
    nbuf = 1 << 14
    tone_bin = 2113
    amp = 7.0
    n = np.arange(-2048, nbuf + 2048)
    e, s_true = _exact_mp_field(n, amp, tone_bin, nbuf)
    intensity = np.abs(e) ** 2
    a, l, _ = O.frontend(intensity, 0.0, v_min=1e-12)
    pos0 = -2048
    jf, jl = -3, (nbuf + 2048 - 768) // 512
    phi = O.hilbert_phase(l, pos0, jf, jl)
    pos = np.arange(512 * jf, 512 * (jl + 1))
    cspr = 10 * np.log10(amp ** 2 / 1.0)
    d = amp ** 2 * (1 + 10 ** (cspr / 10)) / 10 ** (cspr / 10)   # so that A_hat == amp
    a_hat = O.carrier_amplitude(d, cspr)
    assert abs(a_hat - amp) < 1e-12
    theta = O.tone_phase(pos, tone_bin, nbuf)
    es = O.reconstruct_downconvert(a[pos - pos0], phi, a_hat, theta)
    ref = s_true[pos - pos0]
    rel = np.linalg.norm(es - ref) / np.linalg.norm(ref)
    assert rel < 1e-10
    # wrong Hilbert sign or wrong downconversion sign -> O(1) error
    es_bad = O.reconstruct_downconvert(a[pos - pos0], -phi, a_hat, theta)
    assert np.linalg.norm(es_bad - ref) / np.linalg.norm(ref) > 0.3
    es_bad2 = O.reconstruct_downconvert(a[pos - pos0], phi, a_hat, -theta)
    assert np.linalg.norm(es_bad2 - ref) / np.linalg.norm(ref) > 0.3


def test_carrier_only_gives_zero():
    """carrier-only input -> E_s = 0 after carrier removal."""
    nbuf = 4096
    n = np.arange(-1024, nbuf + 1024)
    amp = 5.0
    intensity = np.full(len(n), amp ** 2)
    a, l, _ = O.frontend(intensity, 0.0)
    phi = O.hilbert_phase(l, -1024, -1, 8)
    pos = np.arange(-512, 4608)
    es = O.reconstruct_downconvert(a[pos + 1024], phi, amp, O.tone_phase(pos, 17, nbuf))
    assert np.max(np.abs(es)) < 1e-12


def test_tone_phase_integer_reduction():
    """theta_n is buffer-local: theta(n + N) == theta(n) exactly (reading R7),
    and fast int64 path == exact Python-int path."""
    nbuf = 1 << 22
    pos = np.array([-17152, -1, 0, 1, 12345, nbuf - 1, nbuf, nbuf + 2303])
    t1 = O.tone_phase(pos, 541065, nbuf)
    t2 = O.tone_phase_fast(pos, 541065, nbuf)
    assert np.array_equal(t1, t2)
    assert O.tone_phase([nbuf + 5], 541065, nbuf)[0] == O.tone_phase([5], 541065, nbuf)[0]


# ---------------------------------------------------------------- S4 static EQ + resample
def _overlap_save_fold(e_s, h, nf, keep):
    """Independent frequency-domain formulation (the method's 'pair of FFTs'):
    window FFT, x H (h placed circularly), fold Z_k=(Y_k+Y_{k+nf/2})/2, nf/2 IFFT."""
    H = np.zeros(nf, dtype=np.complex128)
    for t, hv in enumerate(h):
        H[(t - 101) % nf] += hv
    H = np.fft.fft(H)
    margin = (nf - keep) // 2
    out = []
    for start in range(margin, len(e_s) - keep - margin + 1, keep):
        w = e_s[start - margin:start - margin + nf]
        Y = np.fft.fft(w) * H
        Z = 0.5 * (Y[:nf // 2] + Y[nf // 2:])
        z = np.fft.ifft(Z)
        out.append(z[margin // 2:margin // 2 + keep // 2])
    return np.concatenate(out)


@pytest.mark.parametrize("nf,keep", [(1024, 768), (2048, 1536), (2048, 1792)])
def test_static_eq_direct_equals_fold_overlap_save(nf, keep):
    """Reading R5: the frequency-domain EQ with spectral fold is exact LTI
    decimation of the 203-tap FIR, independent of the FFT size."""
    rng = np.random.default_rng(7)
    e_s = rng.standard_normal(8 * keep + nf) + 1j * rng.standard_normal(8 * keep + nf)
    h = rng.standard_normal(203) + 1j * rng.standard_normal(203)
    fs = _overlap_save_fold(e_s, h, nf, keep)
    margin = (nf - keep) // 2
    x2 = O.static_eq_resample(e_s, 0, h, margin // 2, len(fs))
    assert np.max(np.abs(fs - x2)) < 1e-11 * np.max(np.abs(x2))


def test_static_eq_impulse_response():
    """E_s = delta at position 1000 -> x2[m] = h_{2m-1000} (tap index check)."""
    e_s = np.zeros(4000, dtype=np.complex128)
    e_s[1000] = 1.0
    h = np.arange(203) + 1j * np.arange(203)[::-1]
    x2 = O.static_eq_resample(e_s, 0, h, 400, 200)
    for m in range(400, 600):
        i = 2 * m - 1000
        expect = h[i + 101] if -101 <= i <= 101 else 0
        assert x2[m - 400] == expect


# ---------------------------------------------------------------- S5 WL LMS
def test_lms_mu_zero_passthrough():
    """mu = 0, centre-spike taps -> taps unchanged, y = x2[2n]."""
    pts, labs = C.make_standard("QAM16")
    rng = np.random.default_rng(2)
    x2 = rng.standard_normal(1000) + 1j * rng.standard_normal(1000)
    w, g, _, _ = O.wl_lms_update(lambda m: x2[m], 10, 300, [0, 1, 0, 0], [0] * 4, 0.0, pts, 0.1, O.UPD_DD_SOFT)
    assert np.array_equal(w, np.array([0, 1, 0, 0], complex)) and not g.any()
    y = O.wl_apply(x2, 0, 10, 300, w, g)
    assert np.array_equal(y, x2[20:620:2])


def test_lms_pilot_converges_to_least_squares():
    """PILOT mode (paper's training mode) on a noiseless linear +
    conjugate mixing channel converges to the exact inverse (LS solution)."""
    pts, labs = C.make_standard("QAM16")
    rng = np.random.default_rng(4)
    n_sym = 20000
    pat = rng.integers(0, 16, n_sym)
    s = pts[pat]
    # x2 at 2 sps: symbol instants carry 0.9 e^{0.3i} s + 0.1 s*; half instants random
    x2 = np.empty(2 * n_sym + 4, dtype=np.complex128)
    x2[0::2][:n_sym] = 0.9 * np.exp(0.3j) * s + 0.1 * np.conj(s)
    x2[1::2] = 0.05 * (rng.standard_normal(n_sym + 2) + 1j * rng.standard_normal(n_sym + 2))
    x2_at = lambda m: x2[m + 2]  # noqa: E731
    w, g, _, em = O.wl_lms_update(x2_at, 0, n_sym - 2, [0, 1, 0, 0], [0] * 4, 2e-2, pts, 0.0, O.UPD_PILOT, pat, 0)
    y = O.wl_apply(x2, -2, 100, 1000, w, g)
    assert np.max(np.abs(y - s[100:1100])) < 1e-3


def test_lms_widely_linear_beats_strictly_linear():
    """SPEC.md l.393 ablation: input x + 0.1 x* -> the WL taps cancel the
    conjugate term; with g frozen at 0 the residual MSE is much higher."""
    pts, labs = C.make_standard("QAM16")
    rng = np.random.default_rng(6)
    n_sym = 12000
    pat = rng.integers(0, 16, n_sym)
    s = pts[pat]
    x2 = np.zeros(2 * n_sym + 4, dtype=np.complex128)
    x2[0::2][:n_sym] = s + 0.1 * np.conj(s)
    x2_at = lambda m: x2[m + 2]  # noqa: E731
    w, g, _, _ = O.wl_lms_update(x2_at, 0, n_sym - 2, [0, 1, 0, 0], [0] * 4, 1e-2, pts, 0.0, O.UPD_PILOT, pat, 0)
    mse_wl = np.mean(np.abs(O.wl_apply(x2, -2, 200, 2000, w, g) - s[200:2200]) ** 2)
    # strictly linear optimum: best w only (g = 0): LS fit of w on the same data
    xs = x2[0::2][200:2200]
    wl = np.vdot(xs, s[200:2200]) / np.vdot(xs, xs)
    mse_sl = np.mean(np.abs(wl * xs - s[200:2200]) ** 2)
    assert mse_wl < 1e-6 and mse_sl > 1e-3


def test_lms_soft_gate_lipschitz():
    """Reading R10: with the soft gate a 1e-6 relative perturbation of x2 moves
    the resulting taps by O(1e-6), so fp32 GPU taps stay close to
    the fp64 oracle's; the gate fraction is in (0,1) for noisy data."""
    pts, labs = C.make_standard("QAM64")
    rng = np.random.default_rng(8)
    n = 4096
    s = pts[rng.integers(0, 64, n)]
    x2 = np.zeros(2 * n + 4, dtype=np.complex128)
    x2[0::2][:n] = s + 0.05 * (rng.standard_normal(n) + 1j * rng.standard_normal(n))
    x2[1::2] = 0.1 * (rng.standard_normal(n + 2) + 1j * rng.standard_normal(n + 2))
    tau = O.d_min(pts) ** 2 / 4
    pert = x2 * (1 + 1e-6 * rng.standard_normal(len(x2)))
    w1, g1, gated, _ = O.wl_lms_update(lambda m: x2[m + 2], 0, n - 2, [0, 1, 0, 0], [0] * 4, 1e-3, pts, tau, 0)
    w2, g2, _, _ = O.wl_lms_update(lambda m: pert[m + 2], 0, n - 2, [0, 1, 0, 0], [0] * 4, 1e-3, pts, tau, 0)
    assert np.max(np.abs(np.r_[w1 - w2, g1 - g2])) < 1e-5
    assert 0 < gated < n


# ---------------------------------------------------------------- S6 decisions
def test_decide_exact_points_and_tie_break():
    """y = p_k -> k; y = 0 on QAM4 (4-way tie) -> index 0."""
    for name in C.STANDARD:
        pts, _ = C.make_standard(name)
        dec, margin = O.decide(pts, pts)
        assert np.array_equal(dec, np.arange(len(pts)))
        # exact point: distance to its cell boundary = half the nearest-neighbour distance
        dd = np.abs(pts[:, None] - pts[None, :]) + np.eye(len(pts)) * 1e9
        assert np.allclose(margin, dd.min(axis=1) / 2, rtol=0, atol=1e-12)
    pts, _ = C.make_standard("QAM4")
    dec, margin = O.decide(np.array([0j]), pts)
    assert dec[0] == 0 and abs(margin[0]) < 1e-15


def test_decide_margin_is_voronoi_distance():
    """m_n = distance of y to the nearest Voronoi boundary: on a square grid it
    is d_min/2 - max(|dx|, |dy|) for interior points (geometry, not the formula)."""
    pts, _ = C.make_standard("QAM16")
    dm = O.d_min(pts)
    rng = np.random.default_rng(3)
    inner = pts[np.abs(pts.real) < 0.5 * 3 * dm / 2][:1]
    for _ in range(200):
        k = rng.integers(len(pts))
        off = (rng.uniform(-0.45, 0.45) + 1j * rng.uniform(-0.45, 0.45)) * dm
        y = pts[k] + off
        dec, m = O.decide(np.array([y]), pts)
        assert dec[0] == k
        # distance to the nearest boundary among the cell's existing neighbours
        cand = []
        for dx, dy in ((1, 0), (-1, 0), (0, 1), (0, -1)):
            nb = pts[k] + dm * complex(dx, dy)
            if np.min(np.abs(pts - nb)) < 1e-9:
                cand.append(dm / 2 - (off.real * dx + off.imag * dy))
        assert abs(m[0] - min(cand)) < 1e-12
    assert inner.size == 1


def test_decide_random_vs_bruteforce_loop():
    pts, _ = C.make_standard("QAM32")
    rng = np.random.default_rng(9)
    y = 1.3 * (rng.standard_normal(500) + 1j * rng.standard_normal(500))
    dec, _ = O.decide(y, pts)
    for yy, d in zip(y, dec):
        best = min(range(len(pts)), key=lambda k: (abs(yy - pts[k]) ** 2, k))
        assert best == d


# ---------------------------------------------------------------- S7 counts
def test_count_errors_basic():
    """identical -> 0; one symbol wrong by a Gray neighbour -> 1 bit."""
    pts, labs = C.make_standard("QAM16")
    ref = np.arange(16)
    r = O.count_errors(ref, ref, labs)
    assert r["sym_errors"] == 0 and r["bit_errors"] == 0 and r["bits"] == 64
    dec = ref.copy()
    dec[0] = int(np.argmin(np.abs(pts - (pts[0] + O.d_min(pts))) + (np.arange(16) == 0) * 9))
    r = O.count_errors(dec, ref, labs)
    assert r["sym_errors"] == 1 and r["bit_errors"] == 1
    r = O.count_errors(ref, (ref + 8) % 16, labs)
    assert r["bit_errors"] == int(sum(bin(int(labs[i]) ^ int(labs[(i + 8) % 16])).count("1") for i in range(16)))


# ---------------------------------------------------------------- constellations
def test_constellation_invariants_and_gray():
    """SPEC.md l.28-30 invariants; Gray labelling of square QAM (reading R12):
    nearest neighbours differ in exactly one bit; QAM4 = (+-1 +-i)/sqrt2."""
    for name in C.STANDARD:
        p, l = C.make_standard(name)
        C.validate(p, l)
        assert abs(np.mean(np.abs(p) ** 2) - 1) < 1e-12
    p, l = C.make_standard("QAM4")
    assert np.allclose(sorted(p, key=lambda z: (z.real, z.imag)),
                       np.array([-1 - 1j, -1 + 1j, 1 - 1j, 1 + 1j]) / np.sqrt(2))
    for name in ("QAM4", "QAM16", "QAM64", "QAM8"):
        p, l = C.make_standard(name)
        dm = O.d_min(p)
        for i in range(len(p)):
            for j in range(len(p)):
                if i != j and abs(abs(p[i] - p[j]) - dm) < 1e-9:
                    assert bin(int(l[i]) ^ int(l[j])).count("1") == 1


def test_cross_layout_geometry():
    """32 = 6x6 minus 4 corners; 128 = 12x12 minus 16 corners (reading R12)."""
    for name, side, ncorner in (("QAM32", 6, 4), ("QAM128", 12, 16)):
        p, _ = C.make_standard(name)
        g = np.round(p / (O.d_min(p) / 2)).astype(complex)
        lv = sorted(set(g.real.astype(int)))
        assert len(lv) == side and len(set(g.imag.astype(int))) == side
        assert side * side - ncorner == len(set(np.round(g, 6)))


def test_data_files_match_oracle(root):
    """The committed data files (inputs shared by both sides) equal the oracle's
    tables; GS files are valid and have GMI >= the conventional format."""
    from oracle import shaping
    for name in C.STANDARD:
        p, l = C.load(os.path.join(root, "data", "constellations", name + ".txt"))
        p0, l0 = C.make_standard(name)
        assert np.max(np.abs(p - p0)) < 1e-14 and np.array_equal(l, l0)
    for gs, base, snr in (("GS8", "QAM8", 14.0), ("GS128", "QAM128", 20.0)):
        p, l = C.load(os.path.join(root, "data", "constellations", gs + ".txt"))
        p0, l0 = C.make_standard(base)
        order = 10 if len(p) <= 8 else 6
        assert shaping.gmi_awgn(p, l, snr, order) > shaping.gmi_awgn(p0, l0, snr, order)


# ---------------------------------------------------------------- metrics
def test_q_thresholds_and_net_rates():
    """PAPER l.83 thresholds <-> BER; PAPER l.103 net rates."""
    fb = GOLD["fec_ber_derived"]
    fq = GOLD["fec_q_db"]
    for key in ("6.7%", "20%"):
        assert abs(Mx.ber_from_q(fq[key]) / fb[key] - 1) < fb["tol_rel"]
        assert abs(Mx.q_from_ber(Mx.ber_from_q(fq[key])) - fq[key]) < 1e-9
    nr = GOLD["net_rate_gbps"]
    assert round(Mx.net_throughput(64, 1.0, 0.20), 1) == nr["QAM64_20%"]
    assert round(Mx.net_throughput(32, 1.0, 0.067), 1) == nr["QAM32_6.7%"]


def test_closed_form_ber_reductions():
    """Cho-Yoon reduces to Q(sqrt(SNR)) for 4-QAM and to
    [3Q(x)+2Q(3x)-Q(5x)]/4, x = sqrt(SNR/5), for 16-QAM;
    and matches a Monte-Carlo brute force for 64-QAM."""
    for snr_db in (0.0, 6.0, 10.0):
        s = 10 ** (snr_db / 10)
        assert abs(Mx.ber_square_qam_gray(4, s) - Mx.qfunc(np.sqrt(s))) < 1e-15
        x = np.sqrt(s / 5)
        ref16 = (3 * Mx.qfunc(x) + 2 * Mx.qfunc(3 * x) - Mx.qfunc(5 * x)) / 4
        assert abs(Mx.ber_square_qam_gray(16, s) / ref16 - 1) < 1e-12
    pts, labs = C.make_standard("QAM64")
    rng = np.random.default_rng(11)
    snr = 10 ** (16 / 10)
    n = 400000
    idx = rng.integers(0, 64, n)
    y = pts[idx] + np.sqrt(1 / snr / 2) * (rng.standard_normal(n) + 1j * rng.standard_normal(n))
    dec, _ = O.decide(y, pts)
    ber = O.count_errors(dec, idx, labs)["bit_errors"] / (6 * n)
    th = Mx.ber_square_qam_gray(64, snr)
    assert abs(ber - th) < 4 * np.sqrt(th / (6 * n)) + 0.02 * th


# ----------------------------------------------------------------------------
# pre-KK intensity equaliser
# ----------------------------------------------------------------------------
def test_pre_equalize_identity_constant_and_delay():
    from oracle import kk_oracle as O
    rng = np.random.default_rng(11)
    c = rng.integers(-2048, 2048, 4000)
    d = 1234.5
    g = np.zeros(15)
    g[7] = 1.0
    assert np.array_equal(O.pre_equalize(c, d, g), c[7:-7] + d)          # identity
    g2 = np.zeros(15)
    g2[9] = 1.0                                                            # k = +2: v'[n] = v[n - 2]
    assert np.array_equal(O.pre_equalize(c, d, g2), c[5:-9] + d)
    k = np.array([0.1, -0.3, 1.4, -0.3, 0.1])
    assert np.allclose(O.pre_equalize(np.full(50, 7), d, k), (7 + d) * k.sum())  # DC gain


def test_pre_equalize_identity_receive_unchanged():
    """receive() with the identity pre-equaliser equals receive() without it."""
    from oracle import kk_oracle as O
    from synth import configs
    from synth.generate import make_pool, make_stream
    wl = configs.get("C2_n16")
    cfg = wl.link
    pool = make_pool(cfg, 1, cache=False)
    h = np.loadtxt("data/fir/C2_n16.txt")
    fir = h[:, 0] + 1j * h[:, 1]
    left, right = O.required_left(4096) + 8, O.required_right() + 8
    st, off = make_stream(pool, 1, left, right)
    kw = dict(buffer_len=cfg.buffer_len, cspr_db=cfg.cspr_db, dc_offset=pool.dc_offset, fir=fir, points=pool.points,
              labels=pool.labels, tone_bin=cfg.tbin, pattern=pool.pattern)
    a = O.receive(st, off, O.RxParams(**kw))
    g = np.zeros(9)
    g[4] = 1.0
    b = O.receive(st, off, O.RxParams(pre_fir=g, **kw))
    assert np.array_equal(a["decisions"], b["decisions"]) and a["bit_errors"] == b["bit_errors"]
    assert np.max(np.abs(a["y"] - b["y"])) == 0.0


def test_pre_equalizer_lowers_the_bandwidth_error_floor():
    """With a 1 GHz PD/ADC bandwidth (the error-floor mechanism of l.70/l.167)
    the noiseless EVM degrades; the LS-trained pre-KK equaliser (oracle.train.train_prefir,
    trained on the filtered/unfiltered noiseless pair) recovers most of it."""
    from dataclasses import replace
    from oracle import kk_oracle as O
    from oracle import train
    from synth.generate import LinkConfig, make_pool, make_stream
    cfg0 = LinkConfig("QAM16", 14.0, None, "one_sided", 1 << 16, seed_noise=77)
    cfg1 = replace(cfg0, adc_bw_hz=1.0e9)
    p0 = make_pool(cfg0, 1, cache=False)
    p1 = make_pool(cfg1, 1, cache=False)
    h = np.loadtxt("data/fir/C2_n16.txt")
    fir = h[:, 0] + 1j * h[:, 1]
    hp = 7
    left, right = O.required_left(4096) + hp, O.required_right() + hp
    s0, off = make_stream(p0, 1, left, right)
    s1, _ = make_stream(p1, 1, left, right)
    g = train.train_prefir(s1, s0, p1.dc_offset, hp)
    kw = dict(buffer_len=cfg1.buffer_len, cspr_db=cfg1.cspr_db, fir=fir, points=p1.points, labels=p1.labels,
              tone_bin=cfg1.tbin, pattern=p1.pattern)
    sym = p1.points[p1.pattern.astype(np.int64)]

    def evm(st, d, pre):
        o = O.receive(st, off, O.RxParams(dc_offset=d, pre_fir=pre, **kw))
        return 10 * np.log10(np.mean(np.abs(o["y"] - sym) ** 2) / np.mean(np.abs(sym) ** 2))
    e_ideal = evm(s0, p0.dc_offset, None)
    e_bw = evm(s1, p1.dc_offset, None)
    e_eq = evm(s1, p1.dc_offset, g)
    assert e_bw > e_ideal + 3.0          # the roll-off raises the floor
    assert e_eq < e_bw - 3.0             # the pre-KK equaliser removes most of it


def test_frame_sync_fft_equals_direct_sum():
    """oracle.train.frame_sync_corr (FFT form) equals the defining double sum at random
    lags, including lags whose window wraps the pattern period."""
    from oracle import train
    rng = np.random.default_rng(7)
    P, n0, L = 4096, 37, 300
    pts = rng.standard_normal(16) + 1j * rng.standard_normal(16)
    pat = rng.integers(0, 16, P)
    e_pos0 = -8
    e_s = rng.standard_normal(4 * (n0 + L) + 16) + 1j * rng.standard_normal(4 * (n0 + L) + 16)
    c = train.frame_sync_corr(e_s, e_pos0, pts, pat, n0, L)
    for k in (0, 1, 5, P - L - n0 + 3, P - 1, int(rng.integers(P))):
        d = train.frame_sync_direct(e_s, e_pos0, pts, pat, n0, L, k)
        assert abs(c[k] - d) <= 1e-9 * max(1.0, abs(d)), (k, c[k], d)


def test_frame_sync_recovers_known_shift():
    """Symbols of a cyclic pattern sent with a known frame offset s, a fixed phase and AWGN
    at 10 dB: the correlation peak is at s and stands far above the mean sidelobe."""
    from oracle import train
    rng = np.random.default_rng(11)
    P, s, n0, L = 2048, 1234, 16, 512
    pts = np.exp(2j * np.pi * np.arange(16) / 16) * (1 + 0.3 * (np.arange(16) % 2))
    pat = rng.integers(0, 16, P)
    nsym = n0 + L + 8
    tx = pts[pat[(np.arange(nsym) + s) % P]] * np.exp(0.7j)
    tx = tx + 0.3 * (rng.standard_normal(nsym) + 1j * rng.standard_normal(nsym))
    e_s = np.zeros(4 * nsym, dtype=np.complex128)
    e_s[0::4] = tx
    k, ck, mean = train.frame_sync(e_s, 0, pts, pat, n0, L)
    assert k == s
    assert abs(ck) ** 2 > 50 * mean


def test_frame_sync_on_oracle_field():
    """End to end on the oracle's S1-S3 field of a synthetic C2 (16-QAM, noisy) buffer read
    from a point 700 symbols into the stream: frame_sync finds n_off = 700."""
    from oracle import train
    from synth import configs
    from synth.generate import make_pool, make_stream
    cfg = configs.get("C2_n16").link
    pool = make_pool(cfg, 2)
    n = cfg.buffer_len
    left, right = 2048, 2048
    st, off = make_stream(pool, 2, left, right)
    s = 700
    start = off + 4 * s
    window = st[start - left: start + n // 2 + right]
    p = O.RxParams(buffer_len=n, cspr_db=cfg.cspr_db, dc_offset=pool.dc_offset, fir=np.zeros(O.FIR_TAPS),
                   points=pool.points, labels=pool.labels, tone_bin=cfg.tbin)
    e_s, e_pos0 = train.field_after_s3(window, left, p)
    k, ck, mean = train.frame_sync(e_s, e_pos0, pool.points, pool.pattern, 64, 1024)
    assert k == s
    assert abs(ck) ** 2 > 20 * mean


def test_train_fir_recovers_planted_equaliser():
    """oracle.train.train_fir (reading R4: the 203-tap FIR at 4 sps,
    y_n = sum_t h[t] E_s[4n + 101 - t], LS-fitted to the known symbols).  Targets made by
    np.convolve of the oracle's own S1-S3 field with planted random taps: the unregularised
    fit returns those taps to 1e-8 (a transposed or shifted tap index cannot), the
    default-ridge fit reproduces the targets, and a fit one symbol off does not."""
    from oracle import train
    from synth.generate import LinkConfig, make_pool, make_stream
    cfg = LinkConfig("QAM4", 12.0, 7.0, "one_sided", 1 << 15, seed_noise=5)
    pool = make_pool(cfg, 1, cache=False)
    st, off = make_stream(pool, 1, 2048, 2048)
    p = O.RxParams(buffer_len=cfg.buffer_len, cspr_db=cfg.cspr_db, dc_offset=pool.dc_offset,
                   fir=np.zeros(O.FIR_TAPS), points=pool.points, labels=pool.labels, tone_bin=cfg.tbin)
    window = st[: off + 4 * 2048 + 2048]
    e_s, e0 = train.field_after_s3(window, off, p)
    h = np.array([1.0, 1j]) @ np.random.default_rng(3).standard_normal((2, O.FIR_TAPS))
    n0, cnt = 40, 1500
    n = np.arange(n0, n0 + cnt)
    s = np.convolve(e_s, h)[4 * n + O.FIR_HALF - e0]
    h0 = train.train_fir(window, off, p, s, n0, cnt, ridge=0.0)
    assert np.max(np.abs(h0 - h)) <= 1e-8 * np.max(np.abs(h))
    hd = train.train_fir(window, off, p, s, n0, cnt)
    yd = np.convolve(e_s, hd)[4 * n + O.FIR_HALF - e0]
    assert np.linalg.norm(yd - s) <= 1e-6 * np.linalg.norm(s)
    hs = train.train_fir(window, off, p, s, n0 + 1, cnt)
    assert np.max(np.abs(hs - h)) > 0.5 * np.max(np.abs(h))


def test_gmi_4qam_equals_twice_bpsk_capacity():
    """oracle.shaping.gmi_awgn (GS points chosen by GMI on the AWGN channel).
    Gray 4-QAM is two independent BPSK bits, one per dimension, so its GMI is exactly
    2 C_BPSK(a = 1/sqrt 2, sigma^2/2), with C_BPSK = 1 - E log2(1 + exp(-2 a y / s2)),
    y ~ N(a, s2).  That integral is done here by adaptive scipy quadrature, independently of
    the oracle's Gauss-Hermite rule.  The order-40 rule matches to 5e-5 bit; the default
    order 10 is within 5e-3 (its quadrature error, largest near 5 dB)."""
    from scipy import integrate
    from oracle import shaping
    pts, labs = C.make_standard("QAM4")

    def c_bpsk(a, s2):
        def f(y):
            return (np.exp(-(y - a) ** 2 / (2 * s2)) / np.sqrt(2 * np.pi * s2)
                    * np.logaddexp(0.0, -2 * a * y / s2) / np.log(2))
        r = 40 * np.sqrt(s2)
        return 1.0 - integrate.quad(f, a - r, a + r, limit=200, epsabs=1e-13)[0]

    for snr_db in (-5.0, 0.0, 5.0, 10.0, 15.0):
        ref = 2 * c_bpsk(1 / np.sqrt(2), 10 ** (-snr_db / 10) / 2)
        assert abs(shaping.gmi_awgn(pts, labs, snr_db, order=40) - ref) <= 5e-5, snr_db
        assert abs(shaping.gmi_awgn(pts, labs, snr_db) - ref) <= 5e-3, snr_db
    assert abs(shaping.gmi_awgn(pts, labs, 40.0, order=40) - 2.0) <= 1e-9


# ------------------------------------------------------------- carrier amplitude (A.3)
def test_carrier_amplitude_equals_generator_tone():
    """Reading R6 / SURVEY A.3: on a noiseless generated buffer the static carrier
    estimate A_hat = sqrt(d c / (1 + c)) equals the tone the GENERATOR put in, scaled by
    its ADC gain, sqrt(g) * A with A = sqrt(c) (synth.generate._tone): d = g mean(I) and
    mean(I) = 1 + c exactly (unit-power signal, tone on a bin outside the signal band).
    Independently of that formula, the field the chain reconstructs in the tone frame,
    E' = a e^{i phi} (S1 + S2, before the carrier subtraction of S3), has its mean at the
    same sqrt(g) A (the tone is the only DC component of E')."""
    from synth import configs
    from synth.generate import make_pool
    for name in ("C1_n16", "C4_n16"):
        cfg = configs.get(name).link
        pool = make_pool(cfg, 1, cache=False, noiseless=True)
        c = 10 ** (cfg.cspr_db / 10)
        a_gen = math.sqrt(pool.gain) * math.sqrt(c)
        a_hat = O.carrier_amplitude(pool.dc_offset, cfg.cspr_db)
        assert abs(a_hat - a_gen) <= 1e-6 * a_gen, (a_hat, a_gen)   # d is float32
        codes = pool.codes[0]
        n = len(codes)
        win = np.concatenate([codes[-256:], codes, codes[:256]])    # circular halo (periodic buffer)
        a, l, _ = O.frontend(win, pool.dc_offset, 1.0)
        phi = O.hilbert_phase(l, -256, 0, n // 512 - 1)
        e_tf = a[256:256 + n] * np.exp(1j * phi)
        m = np.mean(e_tf)
        assert abs(abs(m) - a_gen) <= 2e-4 * a_gen, (abs(m), a_gen)
        assert abs(np.angle(m)) <= 2e-4
        # the wrong CSPR in the formula is visible: 1 dB off moves A_hat by > 0.1 % (>> 1e-6)
        assert abs(O.carrier_amplitude(pool.dc_offset, cfg.cspr_db + 1.0) - a_gen) > 1e-3 * a_gen


# ------------------------------------------------------------- LMS fixed point (Wiener)
def test_lms_converges_to_wiener_gain():
    """LMS with a known reference (PILOT, the paper's training mode) is a
    stochastic-gradient solver of the Wiener (MMSE) equations: for x2 = s + n at the
    symbol instants (white complex noise, Es/N0 = SNR) and independent noise at the half
    instants, the Wiener taps are w = (0, SNR/(1+SNR), 0, 0), g = 0.  The decision-
    directed soft-gated mode (the default, DD_SOFT) reaches the same fixed point when
    decisions are reliable (4-QAM at 12 dB).  This gain bias is what makes the adaptive
    stage shrink the constellation (C2 BER note)."""
    pts, labs = C.make_standard("QAM4")
    rng = np.random.default_rng(12)
    n_sym = 200000
    snr = 10 ** 1.2
    pat = rng.integers(0, 4, n_sym)
    s = pts[pat]
    sig = math.sqrt(1 / snr / 2)
    x2 = np.empty(2 * n_sym + 4, dtype=np.complex128)
    x2[0::2] = sig * (rng.standard_normal(n_sym + 2) + 1j * rng.standard_normal(n_sym + 2))
    x2[2::2][:n_sym] += s                      # x2_at(2n) = x2[2n + 2] carries s_n (centre tap, index 1)
    x2[1::2] = sig * (rng.standard_normal(n_sym + 2) + 1j * rng.standard_normal(n_sym + 2))
    x2_at = lambda m: x2[m + 2]  # noqa: E731
    wiener = snr / (1 + snr)
    tau = O.d_min(pts) ** 2 / 4
    for mode, t in ((O.UPD_PILOT, 0.0), (O.UPD_DD_SOFT, tau)):
        w, g, _, _ = O.wl_lms_update(x2_at, 0, n_sym - 2, [0, 1, 0, 0], [0] * 4, 2e-4, pts, t, mode, pat, 0)
        assert abs(w[1] - wiener) <= 6e-3, (mode, w)
        assert np.max(np.abs(np.r_[w[[0, 2, 3]], g])) <= 6e-3, (mode, w, g)


# ------------------------------------------------------------- GS optimiser
def test_optimize_recovers_gray_4qam():
    """PAPER l.124 optimiser (oracle.shaping.optimize): started from 4-QAM with a
    non-Gray labelling (diagonal points differ in one bit), the label swaps must find a
    Gray labelling (every pair of nearest neighbours differs in exactly one bit) and the
    GMI must reach Gray 4-QAM's, which is pinned to 2 C_BPSK by independent quadrature
    (test_gmi_4qam_equals_twice_bpsk_capacity); the accepted-GMI trace never decreases."""
    from oracle import shaping
    pts, labs = C.make_standard("QAM4")
    order = np.argsort(np.angle(pts))          # the 4 points counter-clockwise
    bad = np.empty(4, dtype=np.int64)
    bad[order] = [0, 1, 2, 3]                  # natural binary around the square: 1-2 and 3-0 differ in 2 bits
    snr_db = 5.0
    g_gray = shaping.gmi_awgn(pts, labs, snr_db, order=20)
    g_bad = shaping.gmi_awgn(pts, bad, snr_db, order=20)
    assert g_bad < g_gray - 0.05
    p2, l2, trace = shaping.optimize(pts, bad, snr_db, iters=60, seed=3, order=20)
    assert np.all(np.diff(trace) >= 0)
    d = np.abs(p2[:, None] - p2[None, :]) + np.eye(4) * 9
    for k in range(4):
        near = np.argsort(d[k])[:2]
        for j in near:
            assert bin(int(l2[k]) ^ int(l2[j])).count("1") == 1, (l2, k, j)
    assert trace[-1] >= g_gray - 1e-3      # (accepted point moves made before the swap leave a near-square geometry)
    assert trace[-1] <= g_gray + 2e-3   # point moves cannot beat Gray QPSK by more than the quadrature error
