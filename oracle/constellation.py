"""Oracle constellations: conventional QAM tables, file loader, hard decision.

TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import anything under oracle/.  The
product path (paper_2108_07004_b200/) never imports it.

Paper basis
-----------
* PAPER.md l.22 (abstract) and l.31: MP 4/8/16/32/64/128-QAM plus GS-8 / GS-128.
* PAPER.md l.53 (Sec. 2): "The constellation points and bit mapping are uploaded
  to the GPU for the equalizer to make decisions based on a minimum Euclidean
  distance criterion" and "does not rely on specific properties of modulation
  formats such as symmetry".
* The paper prints no coordinates and no bit labels (figures only, PAPER.md
  l.128-159).  Readings (R12):
  Gray labels per axis for square QAM, 8-QAM = 4x2 rectangle with Gray per
  axis, 32/128 = cross layouts obtained by folding the outer columns of an
  8x4 / 16x8 rectangular Gray constellation onto the top/bottom rows.
  Points are normalised to unit mean power.
* Decision rule: argmin_k |y - p_k|^2 with ties to the lowest index
  (reading R11).
"""
from __future__ import annotations

import numpy as np

STANDARD = ("QAM4", "QAM8", "QAM16", "QAM32", "QAM64", "QAM128")


def _gray(i: int) -> int:
    return i ^ (i >> 1)


def _rect(levels_i: int, levels_q: int):
    """Rectangular Gray constellation, index k = iI*levels_q + iQ."""
    bq = int(np.log2(levels_q))
    pts, labs = [], []
    for ii in range(levels_i):
        for iq in range(levels_q):
            pts.append(complex(2 * ii - (levels_i - 1), 2 * iq - (levels_q - 1)))
            labs.append((_gray(ii) << bq) | _gray(iq))
    return np.array(pts, dtype=np.complex128), np.array(labs, dtype=np.int64)


def _cross(levels_i: int, levels_q: int):
    """Cross constellation from a (2L x L) rectangular Gray layout.

    Points with |x| > 1.5*levels_q - 1 (the outer levels_i/8 columns on each
    side) are folded onto the rows above/below the square core:
        x' = sign(x) * (levels_q - |y|),  y' = sign(y) * (|x| - levels_i/4)
    32-QAM: 8x4 -> 6x6 minus corners; 128-QAM: 16x8 -> 12x12 minus corners.
    """
    pts, labs = _rect(levels_i, levels_q)
    core_max = 1.5 * levels_q - 1  # kept columns |x| <= core_max
    shift = levels_i // 4
    out = pts.copy()
    for k, p in enumerate(pts):
        x, y = p.real, p.imag
        if abs(x) > core_max:
            out[k] = complex(np.sign(x) * (levels_q - abs(y)), np.sign(y) * (abs(x) - shift))
    return out, labs


def make_standard(name: str):
    """Return (points complex128 [M], labels int64 [M]) at unit mean power."""
    if name == "QAM4":
        p, l = _rect(2, 2)
    elif name == "QAM8":
        p, l = _rect(4, 2)
    elif name == "QAM16":
        p, l = _rect(4, 4)
    elif name == "QAM32":
        p, l = _cross(8, 4)
    elif name == "QAM64":
        p, l = _rect(8, 8)
    elif name == "QAM128":
        p, l = _cross(16, 8)
    else:
        raise ValueError(f"unknown format {name}")
    p = p / np.sqrt(np.mean(np.abs(p) ** 2))
    return p, l


def validate(points, labels):
    """SPEC.md l.28-30 invariants: M power of two, 4<=M<=128, labels a bijection."""
    m = len(points)
    if m < 4 or m > 128 or (m & (m - 1)):
        raise ValueError("M must be a power of two in [4, 128]")
    if len(labels) != m or sorted(int(x) for x in labels) != list(range(m)):
        raise ValueError("labels must enumerate all log2(M)-bit strings once")


def load(path: str):
    """SPEC.md l.89 text format: '<re> <im> <bitlabel>' per line, '#' comments.

    Normalisation to unit mean power is applied on load."""
    pts, labs = [], []
    with open(path) as f:
        for line in f:
            line = line.split("#", 1)[0].strip()
            if not line:
                continue
            re_, im_, lab = line.split()
            pts.append(complex(float(re_), float(im_)))
            labs.append(int(lab, 2))
    p = np.array(pts, dtype=np.complex128)
    l = np.array(labs, dtype=np.int64)
    validate(p, l)
    p = p / np.sqrt(np.mean(np.abs(p) ** 2))
    return p, l


def save(path: str, points, labels, comment: str = ""):
    m = len(points)
    b = int(np.log2(m))
    with open(path, "w") as f:
        if comment:
            for c in comment.splitlines():
                f.write(f"# {c}\n")
        for p, l in zip(points, labels):
            f.write(f"{p.real:+.17e} {p.imag:+.17e} {int(l):0{b}b}\n")


def demap_hard(y, points):
    """argmin_k |y - p_k|^2, ties -> lowest k. Brute force."""
    y = np.atleast_1d(np.asarray(y, dtype=np.complex128))
    d = np.abs(y[:, None] - points[None, :]) ** 2
    return np.argmin(d, axis=1)  # np.argmin returns the first (lowest) index on ties


def min_distance(points) -> float:
    d = np.abs(points[:, None] - points[None, :])
    d[np.arange(len(points)), np.arange(len(points))] = np.inf
    return float(d.min())
