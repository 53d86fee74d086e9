"""End-to-end pins of the oracle chain (S1-S7) on synthetic workloads.

* noiseless back-to-back -> zero errors (SPEC.md l.400 / l.606)
* one-sided AWGN: BER equals the Gray square-QAM closed form at the realised
  Es/N0 (Cho-Yoon; 4-QAM = Q(sqrt(SNR))) -- with mu = 0 the chain is
  KK + matched filter + slicer, so a dropped term or sign error anywhere shows.
"""
import os

import numpy as np
import pytest

from oracle import kk_oracle as O
from oracle import metrics as Mx
from oracle import train
from synth import configs
from synth.generate import LinkConfig, make_pool, make_stream, noise_psd

LEFT = O.required_left(4096)
RIGHT = 2304


def _fir(name):
    h = np.loadtxt(f"data/fir/{name}.txt")
    return h[:, 0] + 1j * h[:, 1]


def _params(pool, cfg, fir, **kw):
    return O.RxParams(buffer_len=cfg.buffer_len, cspr_db=cfg.cspr_db, dc_offset=pool.dc_offset, fir=fir,
                      points=pool.points, labels=pool.labels, tone_bin=cfg.tbin, pattern=pool.pattern, **kw)


def test_noiseless_back_to_back_zero_errors(root):
    wl = configs.get("C1_n16")
    pool = make_pool(wl.link, 1, cache=False)
    st, off = make_stream(pool, 1, LEFT, RIGHT)
    r = O.receive(st, off, _params(pool, wl.link, _fir("C1_n16")))
    assert r["sym_errors"] == 0 and r["bit_errors"] == 0
    assert np.array_equal(r["decisions"], pool.pattern[: wl.link.n_sym].astype(np.int64))
    sym = pool.points[pool.pattern[: wl.link.n_sym].astype(np.int64)]
    evm_db = 10 * np.log10(np.mean(np.abs(r["y"] - sym) ** 2))
    assert evm_db < -35.0
    assert r["margin"].min() > 1e-2  # exempt set empty -> totals must be bit-identical


def test_one_sided_awgn_16qam_closed_form(root):
    wl = configs.get("C2_n16")
    cfg = wl.link
    pool = make_pool(cfg, 8, cache=False)
    fir = _fir("C2_n16")
    errs = bits = 0
    for b in range(8):
        st, off = make_stream(pool, 1, LEFT, RIGHT, first=b)
        r = O.receive(st, off, _params(pool, cfg, fir, mu=0.0))
        errs += r["bit_errors"]
        bits += r["bits"]
    th = Mx.ber_square_qam_gray(16, 1.0 / (noise_psd(cfg) * 1e9))
    ber = errs / bits
    assert abs(ber - th) <= 3 * np.sqrt(th / bits) + 0.02 * th, (ber, th)


def test_one_sided_awgn_4qam_q_function():
    """4-QAM BER = Q(sqrt(Es/N0)); static EQ trained in-test
    with oracle.train on the noiseless twin."""
    cfg = LinkConfig("QAM4", 12.0, 7.0, "one_sided", 1 << 17, seed_noise=77)
    pool0 = make_pool(cfg, 1, cache=False, noiseless=True)
    st0, off0 = make_stream(pool0, 1, 2048, 2048)
    sym = pool0.points[pool0.pattern.astype(np.int64)]
    p0 = _params(pool0, cfg, np.zeros(203))
    fir = train.train_fir(st0[: off0 + 4 * 8192 + 2048], off0, p0, sym[:8192], 0, 8192)
    pool = make_pool(cfg, 2, cache=False)
    errs = bits = 0
    for b in range(2):
        st, off = make_stream(pool, 1, LEFT, RIGHT, first=b)
        r = O.receive(st, off, _params(pool, cfg, fir, mu=0.0))
        errs += r["bit_errors"]
        bits += r["bits"]
    snr = 1.0 / (noise_psd(cfg) * 1e9)
    th = float(Mx.qfunc(np.sqrt(snr)))
    ber = errs / bits
    assert abs(ber - th) <= 3 * np.sqrt(th / bits) + 0.02 * th, (ber, th)
    # the adaptive equaliser in its default DD-soft mode converges and costs < 0.2 dB
    st, off = make_stream(pool, 1, LEFT, RIGHT, first=0)
    r = O.receive(st, off, _params(pool, cfg, fir))
    assert r["bit_errors"] / r["bits"] < float(Mx.qfunc(np.sqrt(snr * 10 ** (-0.02))))  + 4 * np.sqrt(th / r["bits"])


def test_window_halo_independence():
    """Outputs depend only on the raw window (SURVEY 8(b) determinism):
    a larger halo gives bit-identical decisions and taps."""
    wl = configs.get("C2_n16")
    pool = make_pool(wl.link, 2, cache=False)
    fir = _fir("C2_n16")
    st, off = make_stream(pool, 1, LEFT, RIGHT, first=1)
    st2, off2 = make_stream(pool, 1, LEFT + 4096, RIGHT + 512, first=1)
    r1 = O.receive(st, off, _params(pool, wl.link, fir))
    r2 = O.receive(st2, off2, _params(pool, wl.link, fir))
    assert np.array_equal(r1["decisions"], r2["decisions"])
    assert np.array_equal(r1["taps"][0][0], r2["taps"][0][0])


def test_window_too_small_raises():
    wl = configs.get("C1_n16")
    pool = make_pool(wl.link, 1, cache=False)
    st, off = make_stream(pool, 1, 1000, RIGHT)
    with pytest.raises(ValueError):
        O.receive(st, off, _params(pool, wl.link, _fir("C1_n16")))


# ------------------------------------------------------------- full-size configs
def _receive_full(args):
    """Worker: oracle.receive on stream buffer b of a full-size workload (fork-started)."""
    name, b, mu = args
    cfg = configs.get(name).link
    pool = make_pool(cfg, _FULL_POOLS[name])
    st, off = make_stream(pool, 1, LEFT, RIGHT, first=b)
    r = O.receive(st, off, _params(pool, cfg, _fir(name), mu=mu))
    sym = pool.points[pool.pattern[: cfg.n_sym].astype(np.int64)]
    g = np.vdot(sym, r["y"]) / np.vdot(sym, sym)
    return r["bit_errors"], r["bits"], g, float(np.mean(np.abs(r["y"] - g * sym) ** 2))


_FULL_POOLS = {"C2": 4, "C4": 16}


def _full_size_run(name, mu):
    import multiprocessing as mp
    cfg = configs.get(name).link
    nb = _FULL_POOLS[name]
    make_pool(cfg, nb)  # generate (and cache) once before the workers read it
    with mp.get_context("fork").Pool(min(8, os.cpu_count() or 1)) as workers:
        res = workers.map(_receive_full, [(name, b, mu) for b in range(nb)])
    errs = sum(r[0] for r in res)
    bits = sum(r[1] for r in res)
    gain = np.mean([r[2] for r in res])
    snr = np.mean([abs(r[2]) ** 2 for r in res]) / np.mean([r[3] for r in res])  # unit-power symbols
    return errs, bits, gain, snr


@pytest.mark.slow
def test_one_sided_awgn_16qam_closed_form_full_size():
    """C2 at its stated size (2^22-sample buffers, 4 of them = 16.8 M bits, mu = 0):
    (i) the realised Es/N0 at the slicer (unbiased: error after removing the fitted
    gain) is within 0.05 dB of the generator's nominal OSNR-derived Es/N0, and the gain
    is 1 within 1e-3 (the unbiased static EQ, reading R4); (ii) the BER equals the
    Gray 16-QAM closed form (Cho-Yoon) AT that realised Es/N0 within 3 sigma + 1 %
    (3 sigma = 2.7 % here), i.e. the KK chain leaves Gaussian-like decision noise."""
    cfg = configs.get("C2").link
    errs, bits, gain, snr = _full_size_run("C2", 0.0)
    nominal = Mx.snr_one_sided(cfg.osnr_db, cfg.cspr_db)
    assert abs(10 * np.log10(snr) - nominal) <= 0.05, (10 * np.log10(snr), nominal)
    assert abs(gain - 1.0) <= 1e-3, gain
    th = Mx.ber_square_qam_gray(16, snr)
    ber = errs / bits
    assert abs(ber - th) <= 3 * np.sqrt(th / bits) + 0.01 * th, (ber, th)


@pytest.mark.slow
def test_c4_hdfec_threshold_full_size():
    """BASELINE config 4 / PAPER l.85: 64-QAM at CSPR 16 dB and OSNR 28.2 dB crosses the
    20 % HD-FEC threshold Q = 6.70 dB -- the chain (default DD_SOFT
    adaptive stage) must reach Q >= 6.70 dB on 16 distinct full-size two-sided-noise
    buffers (100 M bits), at a realised Es/N0 within 0.3 dB of the two-sided
    prediction (20.05 dB)."""
    cfg = configs.get("C4").link
    errs, bits, gain, snr = _full_size_run("C4", 1e-3)
    q = float(Mx.q_from_ber(errs / bits))
    assert q >= Mx.FEC_THRESHOLDS_DB["20%"], q
    pred = Mx.snr_two_sided(cfg.osnr_db, cfg.cspr_db)
    assert abs(10 * np.log10(snr) - pred) <= 0.3, (10 * np.log10(snr), pred)
