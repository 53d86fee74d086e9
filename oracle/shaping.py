"""GMI evaluation and the GS optimiser of PAPER.md Sec. 5 (used to produce the
committed GS-8 / GS-128 data files).

TEST / TOOL INFRASTRUCTURE ONLY (see oracle/kk_oracle.py header).

PAPER l.124: "The constellations are initialized using the conventional layout
and optimized by iterating between adding perturbations in the form of Gaussian
noise to a randomly chosen single point and swapping the binary labels of two
randomly chosen constellation points until convergence is reached. After each
iteration, the GMI for the AWGN channel is evaluated and if gains are found,
the modified constellation is taken as the new baseline."  "Symmetries are added
to GS-128-QAM to aid convergence."

Parity unpinned: the optimised GS-8 / GS-128 *geometry* that
optimize() produces -- the paper prints no coordinates; only unit power, bijective
labels, GMI >= the conventional layout and the Gray 4-QAM recovery are pinned.
gmi_awgn itself is pinned (Gray 4-QAM = 2 x BPSK AWGN capacity).

GMI: standard BICM generalised mutual information, complex AWGN
with Es = 1, N0 = 1/SNR, expectation by 2-D Gauss-Hermite quadrature.
"""
from __future__ import annotations

import numpy as np


def gmi_awgn(points, labels, snr_db, order=10):
    points = np.asarray(points, dtype=np.complex128)
    labels = np.asarray(labels, dtype=np.int64)
    m = len(points)
    nb = int(np.log2(m))
    sigma2 = 10 ** (-snr_db / 10)
    t, w = np.polynomial.hermite.hermgauss(order)
    nr, ni = np.meshgrid(t, t, indexing="ij")
    noise = np.sqrt(sigma2) * (nr + 1j * ni).reshape(-1)       # CN(0, sigma2)
    wts = (np.outer(w, w) / np.pi).reshape(-1)
    y = points[:, None] + noise[None, :]                         # [M, Q]
    d = np.abs(y[:, :, None] - points[None, None, :]) ** 2       # [M, Q, M]
    logp = -d / sigma2
    mx = logp.max(axis=2, keepdims=True)
    p = np.exp(logp - mx)
    den = p.sum(axis=2)                                          # [M, Q]
    total = 0.0
    for i in range(nb):
        bit = (labels >> i) & 1                                  # [M]
        same = bit[None, None, :] == bit[:, None, None]          # [M, 1, M]
        num = np.where(same, p, 0.0).sum(axis=2)                 # [M, Q]
        total += np.sum(wts[None, :] * np.log2(den / num)) / m
    return nb - total


def optimize(points, labels, snr_db, iters=2000, seed=0, sym4=False, step=0.05, order=10):
    """Alternate Gaussian perturbation of one point and a label swap of two
    points; accept iff GMI strictly improves.  With sym4, the
    point set is kept invariant under 90-degree rotation (perturbation moves
    all four images; labels of images differ only in the 2 quadrant MSBs)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    pts = np.asarray(points, dtype=np.complex128).copy()
    labs = np.asarray(labels, dtype=np.int64).copy()
    m = len(pts)
    best = gmi_awgn(pts, labs, snr_db, order)
    trace = [best]
    dmin0 = np.min(np.abs(pts[:, None] - pts[None, :]) + np.eye(m) * 1e9)
    sd = step * dmin0
    rejects = 0
    if sym4:
        # orbit of index k under rotation by j: the point with p_k * 1j**j
        orb = np.zeros((m, 4), dtype=np.int64)
        for k in range(m):
            for j in range(4):
                orb[k, j] = int(np.argmin(np.abs(pts - pts[k] * (1j ** j))))
    for it in range(iters):
        cand_p, cand_l = pts.copy(), labs.copy()
        if it % 2 == 0:
            k = rng.integers(m)
            delta = sd * (rng.standard_normal() + 1j * rng.standard_normal())
            if sym4:
                for j in range(4):
                    cand_p[orb[k, j]] = cand_p[orb[k, j]] + delta * (1j ** j)
            else:
                cand_p[k] += delta
            cand_p /= np.sqrt(np.mean(np.abs(cand_p) ** 2))
        else:
            a, b = rng.choice(m, 2, replace=False)
            if sym4:
                for j in range(4):
                    ia, ib = orb[a, j], orb[b, j]
                    if ia == ib:
                        continue
                    la, lb = cand_l[ia], cand_l[ib]
                    cand_l[ia], cand_l[ib] = lb, la
                if len(set(cand_l.tolist())) != m:
                    continue
            else:
                cand_l[a], cand_l[b] = cand_l[b], cand_l[a]
        g = gmi_awgn(cand_p, cand_l, snr_db, order)
        if g > best:
            pts, labs, best = cand_p, cand_l, g
            rejects = 0
        else:
            rejects += 1
            if rejects % 200 == 0:
                sd *= 0.5
        trace.append(best)
    return pts, labs, np.array(trace)
