"""Exactness of the two decision look-up tables of libkkrx.so (host-built, no GPU).

The fused chain's decision (S6) and the LMS update pass (S5) both replace the
brute-force minimum-distance search of the oracle (oracle.kk_oracle.decide;
PAPER.md l.47 "symbol decision", SPEC.md l.65-73 ties -> lowest index) by a
per-cell candidate list.  These tests pin the tables against brute force over
all points on dense random and boundary-hugging samples, for every format:

* chain table (4 candidates): the argmin over the cell's list == brute-force
  argmin (lowest index on ties) for every y inside the grid;
* LMS table: FAST cells => that point is the brute-force nearest and every other
  point is >= tau farther (soft gate gamma = 1); SLOW cells => the list holds the
  nearest point and every point within tau of it, so k1, D1 and the gated D2 of
  the oracle follow exactly from the list.
"""
import ctypes as C

import numpy as np
import pytest

from paper_2108_07004_b200 import _lib
from synth.generate import load_constellation

FORMATS = ["QAM4", "QAM8", "QAM16", "QAM32", "QAM64", "QAM128", "GS8", "GS128"]


def _tables(pts, tau):
    lib = _lib.load()
    m = len(pts)
    pf = np.ascontiguousarray(np.stack([pts.real, pts.imag], -1).reshape(-1).astype(np.float32))
    G = 128
    lms = np.zeros(2 * G * G, np.float32)
    lg = np.zeros(3, np.float32)
    dec = np.zeros(128 * 128, np.uint32)
    dg = np.zeros(4, np.float32)
    fp = C.POINTER(C.c_float)
    r = lib.kk_rx_decision_tables(pf.ctypes.data_as(fp), m, float(tau), lms.ctypes.data_as(fp), lg.ctypes.data_as(fp),
                                  dec.ctypes.data_as(C.POINTER(C.c_uint32)), dg.ctypes.data_as(fp))
    assert r == G
    return pf.reshape(-1, 2), lms.reshape(G * G, 2), lg, dec, dg


def _samples(pts32, n, seed):
    """Uniform over the bounding box (+margin) plus points hugging Voronoi boundaries."""
    rng = np.random.default_rng(seed)
    p = pts32[:, 0] + 1j * pts32[:, 1]
    lo = min(p.real.min(), p.imag.min()) - 0.3
    hi = max(p.real.max(), p.imag.max()) + 0.3
    u = rng.uniform(lo, hi, n) + 1j * rng.uniform(lo, hi, n)
    i = rng.integers(0, len(p), n)
    j = rng.integers(0, len(p), n)
    t = 0.5 + rng.normal(0, 0.02, n)
    mid = p[i] + t * (p[j] - p[i]) + rng.normal(0, 1e-3, n) * (1 + 1j)
    y = np.concatenate([u, mid])
    return y.real.astype(np.float32), y.imag.astype(np.float32)


def _brute(pts32, yx, yy):
    d = (yx[:, None].astype(np.float64) - pts32[None, :, 0]) ** 2 + (yy[:, None].astype(np.float64) - pts32[None, :, 1]) ** 2
    k1 = np.argmin(d, axis=1)                        # lowest index on ties
    ds = np.sort(d, axis=1)
    return k1, ds[:, 0], ds[:, 1] if d.shape[1] > 1 else np.full(len(yx), np.inf), d


@pytest.mark.parametrize("fmt", FORMATS)
def test_chain_decision_table_equals_brute_force(fmt):
    pts, _ = load_constellation(fmt)
    pts32, _, _, dec, dg = _tables(pts, 0.0)
    g = int(dg[3])
    yx, yy = _samples(pts32, 40000, 1)
    k1, _, _, d = _brute(pts32, yx, yy)
    if g == 0:
        assert len(pts) <= 8
        return
    fx = (yx - np.float32(dg[0])) * np.float32(dg[2])
    fy = (yy - np.float32(dg[1])) * np.float32(dg[2])
    inside = (fx >= 0) & (fy >= 0) & (fx < g) & (fy < g)
    w = dec[(np.clip(fy, 0, g - 1).astype(np.int64) * g + np.clip(fx, 0, g - 1).astype(np.int64))]
    use = inside & ((w >> 31) == 0)
    assert use.mean() > 0.5
    cand = np.stack([(w >> (7 * c)) & 127 for c in range(4)], 1).astype(np.int64)
    dc = np.take_along_axis(d, cand, 1)
    # ascending candidates + first minimum == lowest index on ties
    got = cand[np.arange(len(cand)), np.argmin(dc, axis=1)]
    assert np.array_equal(got[use], k1[use])


@pytest.mark.parametrize("fmt", FORMATS)
@pytest.mark.parametrize("gate", ["soft", "hard"])
def test_lms_table_fast_and_slow_cells(fmt, gate):
    pts, _ = load_constellation(fmt)
    p = pts
    dd = np.abs(p[:, None] - p[None, :])
    tau = float(dd[dd > 0].min() ** 2 / 4) if gate == "soft" else 0.0
    pts32, lms, lg, _, _ = _tables(pts, tau)
    G = 128
    yx, yy = _samples(pts32, 60000, 2)
    k1, d1, d2, d = _brute(pts32, yx, yy)
    fx = np.clip(yx * lg[2] + lg[0], 0, G - 1).astype(np.int64)
    fy = np.clip(yy * lg[2] + lg[1], 0, G - 1).astype(np.int64)
    ent = lms[fy * G + fx]
    fast = ~np.isnan(ent[:, 0])
    assert fast.mean() > 0.3
    # FAST: the stored point is the nearest and the gate is open (D2 - D1 >= tau)
    kf = k1[fast]
    assert np.array_equal(ent[fast, 0], pts32[kf, 0]) and np.array_equal(ent[fast, 1], pts32[kf, 1])
    assert np.all(d2[fast] - d1[fast] >= tau * (1 - 1e-6))
    # SLOW: list (ascending, 128-padded) holds the nearest and every point within tau of it
    wbits = ent[~fast, 1].view(np.uint32)
    brute = wbits == 0xFFFFFFFF
    lst = np.stack([(wbits >> (8 * c)) & 0xFF for c in range(4)], 1).astype(np.int64)
    valid = lst < 128
    assert np.all(np.diff(np.where(valid, lst, 1000), axis=1)[valid[:, 1:]] > 0)   # ascending
    ds = d[~fast]
    near = ds <= (d1[~fast] + tau)[:, None]
    for r in np.nonzero(~brute)[0][:20000]:
        need = np.nonzero(near[r])[0]
        have = set(lst[r][valid[r]].tolist())
        assert set(need.tolist()) <= have, (r, need, have)
    # outer ring of cells is brute force (receives every clamped y)
    ring = np.zeros((G, G), bool)
    ring[0, :] = ring[-1, :] = ring[:, 0] = ring[:, -1] = True
    rb = lms.reshape(G, G, 2)[ring]
    assert np.all(np.isnan(rb[:, 0])) and np.all(rb[:, 1].view(np.uint32) == 0xFFFFFFFF)
