"""Oracle metrics: Q factor, HD-FEC thresholds, net throughput, closed-form BER.

TEST INFRASTRUCTURE ONLY (see oracle/kk_oracle.py header).

* Q = 20 log10(sqrt(2) erfcinv(2 BER))  -- reading R13; the paper
  quotes Q thresholds 8.35 dB (6.7 % OH) and 6.70 dB (20 % OH).
* Net rate = baud * log2(M) / (1 + OH)  -- PAPER.md l.103 (5 Gbps 64-QAM 20 %,
  4.7 Gbps 32-QAM 6.7 %).
* Closed-form Gray square-QAM BER in AWGN: Cho & Yoon (2002) exact expression;
  4-QAM reduces to Q(sqrt(SNR)).  Used to pin the oracle chain end to end on
  one-sided AWGN.
"""
from __future__ import annotations

import math

import numpy as np
from scipy.special import erfc, erfcinv

FEC_THRESHOLDS_DB = {"6.7%": 8.35, "20%": 6.70}
FEC_OVERHEAD = {"6.7%": 0.067, "20%": 0.20}


def q_from_ber(ber):
    ber = np.asarray(ber, dtype=np.float64)
    return 20.0 * np.log10(np.sqrt(2.0) * erfcinv(2.0 * ber))


def ber_from_q(q_db):
    q = 10.0 ** (np.asarray(q_db, dtype=np.float64) / 20.0)
    return 0.5 * erfc(q / np.sqrt(2.0))


def net_throughput(m, baud, overhead):
    return baud * math.log2(m) / (1.0 + overhead)


def qfunc(x):
    return 0.5 * erfc(np.asarray(x, dtype=np.float64) / np.sqrt(2.0))


def ber_square_qam_gray(m, snr_lin):
    """Exact BER of Gray-labelled square M-QAM in complex AWGN, Es/N0 = snr_lin.

    Cho & Yoon, IEEE Trans. Commun. 50(7), 2002, eq. (14)-(16)."""
    sm = int(round(math.sqrt(m)))
    assert sm * sm == m
    nb = int(round(math.log2(sm)))
    total = 0.0
    for k in range(1, nb + 1):
        acc = 0.0
        for i in range(int((1 - 2.0 ** (-k)) * sm)):
            w = (-1) ** math.floor(i * 2 ** (k - 1) / sm) * (2 ** (k - 1) - math.floor(i * 2 ** (k - 1) / sm + 0.5))
            acc += w * erfc((2 * i + 1) * math.sqrt(3.0 * snr_lin / (2.0 * (m - 1))))
        total += acc / sm
    return total / nb


def snr_one_sided(osnr_db, cspr_db, baud=1e9, ref_bw=12.5e9):
    """Es/N0 (dB) for the one-sided noise mode: noise PSD N0 with
    N0 * 12.5 GHz = P_total 10^(-OSNR/10), P_total = P_s (1 + c)."""
    c = 10 ** (cspr_db / 10)
    return osnr_db + 10 * math.log10(ref_bw / baud) - 10 * math.log10(1 + c)


def snr_two_sided(osnr_db, cspr_db, baud=1e9, ref_bw=12.5e9):
    """Predicted Es/N0 (dB) after KK detection for the two-sided (physical) noise mode:
    the ASE is flat on both sides of the tone, so the image-band noise beats with the
    carrier onto the same baseband frequencies as the signal-band noise and the
    in-band noise doubles: snr_one_sided - 10 log10(2) (SURVEY.md 8(c) reading 14)."""
    return snr_one_sided(osnr_db, cspr_db, baud, ref_bw) - 10 * math.log10(2.0)
