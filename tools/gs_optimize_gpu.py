"""Geometric-shaping optimiser on the GPU.

The paper's loop: perturb one point by Gaussian noise or swap the labels of two points,
evaluate the AWGN GMI, keep the move iff the GMI improves.  Here every iteration draws
B candidate moves (B = 1 is exactly the paper's loop) and evaluates them in ONE batched
kk_gmi_awgn launch (one CTA per candidate), keeping the best strictly improving one.
Optional quadrant symmetry (90-degree rotations, as for GS-128, "symmetries are added to
aid convergence") as in oracle/shaping.py.  The random moves are drawn on the host
(PCG64, seeded) and passed in as data.

    python tools/gs_optimize_gpu.py --fmt QAM128 --snr 20 --order 6 --iters 200 --batch 64 --sym4
    python tools/gs_optimize_gpu.py --fmt QAM8 --snr 14 --iters 400 --batch 32 [--write GS8_gpu.txt]

Prints the GMI trace, the GMI of the committed GS table for comparison, and wall time.
"""
import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2108_07004_b200 import gmi_awgn  # noqa: E402
from synth.generate import load_constellation  # noqa: E402


def orbits(pts):
    m = len(pts)
    orb = np.zeros((m, 4), dtype=np.int64)
    for k in range(m):
        for j in range(4):
            orb[k, j] = int(np.argmin(np.abs(pts - pts[k] * (1j ** j))))
    return orb


def propose(rng, pts, labs, sd, sym4, orb, kind):
    p, l = pts.copy(), labs.copy()
    m = len(p)
    if kind == 0:
        k = rng.integers(m)
        delta = sd * (rng.standard_normal() + 1j * rng.standard_normal())
        if sym4:
            for j in range(4):
                p[orb[k, j]] += delta * (1j ** j)
        else:
            p[k] += delta
        p /= np.sqrt(np.mean(np.abs(p) ** 2))
    else:
        a, b = rng.choice(m, 2, replace=False)
        if sym4:
            for j in range(4):
                ia, ib = orb[a, j], orb[b, j]
                if ia != ib:
                    l[ia], l[ib] = l[ib], l[ia]
            if len(set(l.tolist())) != m:
                return None
        else:
            l[a], l[b] = l[b], l[a]
    return p, l


def optimize_gpu(pts, labs, snr_db, iters=300, batch=32, sym4=False, seed=1, step=0.05, order=10):
    """The paper's perturb/swap loop with `batch` candidate moves per batched
    kk_gmi_awgn launch (batch = 1: the paper's loop, one move per GMI evaluation).  Returns
    (points, labels, GMI trace of the accepted baseline, first entry = the start)."""
    pts = np.asarray(pts, dtype=np.complex128)
    pts = pts / np.sqrt(np.mean(np.abs(pts) ** 2))
    labs = np.asarray(labs, dtype=np.int64).copy()
    rng = np.random.Generator(np.random.PCG64(seed))
    orb = orbits(pts) if sym4 else None
    m = len(pts)
    dmin = np.min(np.abs(pts[:, None] - pts[None, :]) + np.eye(m) * 1e9)
    sd = step * dmin
    best = float(np.atleast_1d(gmi_awgn(pts, labs, snr_db, order))[0])
    trace = [best]
    stall = 0
    for it in range(iters):
        cands = []
        while len(cands) < batch:
            # batch = 1 alternates perturbation / swap over the iterations like the oracle loop
            c = propose(rng, pts, labs, sd, sym4, orb, kind=(len(cands) if batch > 1 else it) % 2)
            if c is not None:
                cands.append(c)
        P = np.stack([c[0] for c in cands])
        L = np.stack([c[1] for c in cands])
        g = np.atleast_1d(gmi_awgn(P, L, snr_db, order))
        k = int(np.argmax(g))
        if g[k] > best:
            pts, labs, best = P[k], L[k], float(g[k])
            stall = 0
        else:
            stall += 1
            if stall % 20 == 0:
                sd *= 0.5
        trace.append(best)
    return pts, labs, np.array(trace)


def write_constellation(path, pts, labs, header):
    """SPEC.md l.89 constellation file: '<re> <im> <label bits>' per point, labels as
    zero-padded binary strings of log2(M) bits (what synth.generate.load_constellation reads)."""
    m = len(pts)
    nbits = int(round(np.log2(m)))
    assert 1 << nbits == m and sorted(int(x) for x in labs) == list(range(m)), "labels must be a bijection on [0, M)"
    with open(path, "w") as f:
        for line in str(header).splitlines():
            f.write(f"# {line}\n")
        for p, l in zip(pts, labs):
            f.write(f"{p.real:+.17e} {p.imag:+.17e} {int(l):0{nbits}b}\n")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--fmt", default="QAM8")
    ap.add_argument("--snr", type=float, default=14.0)
    ap.add_argument("--order", type=int, default=10)
    ap.add_argument("--iters", type=int, default=300)
    ap.add_argument("--batch", type=int, default=32)
    ap.add_argument("--sym4", action="store_true")
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--step", type=float, default=0.05)
    ap.add_argument("--write", default="")
    a = ap.parse_args()
    pts, labs = load_constellation(a.fmt)
    t0 = time.time()
    pts, labs, trace = optimize_gpu(pts, labs, a.snr, a.iters, a.batch, a.sym4, a.seed, a.step, a.order)
    dt = time.time() - t0
    g0, best = trace[0], trace[-1]
    ref = {"QAM8": "GS8", "QAM128": "GS128"}.get(a.fmt)
    line = f"{a.fmt} @ {a.snr} dB: GMI {g0:.5f} -> {best:.5f} bits in {a.iters} iterations x {a.batch} candidates, " \
           f"{dt:.1f} s ({a.iters * a.batch / dt:.0f} GMI evaluations/s on the GPU)"
    if ref:
        rp, rl = load_constellation(ref)
        line += f"; committed {ref}: {float(np.atleast_1d(gmi_awgn(rp, rl, a.snr, a.order))[0]):.5f}"
    print(line)
    if a.write:
        write_constellation(a.write, pts, labs, f"GS from tools/gs_optimize_gpu.py {vars(a)}  GMI {best:.6f}")


if __name__ == "__main__":
    main()
