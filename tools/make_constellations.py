"""Write data/constellations/*.txt (SPEC.md l.89 format) using only oracle/.

Conventional formats come from oracle.constellation.make_standard (readings R12).
GS-8 (14 dB) and GS-128 (20 dB) come from oracle.shaping.optimize with a fixed
seed.  The paper prints no GS coordinates, so the GS geometry
is a committed choice ("parity unpinned" for the geometry itself; checks: unit
power, bijective labels, GMI >= conventional at the target SNR).

Run:  python tools/make_constellations.py [--gs-iters 3000 --gs128-iters 800]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from oracle import constellation as C  # noqa: E402
from oracle import shaping  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "data", "constellations")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gs8-iters", type=int, default=3000)
    ap.add_argument("--gs128-iters", type=int, default=600)
    a = ap.parse_args()
    os.makedirs(OUT, exist_ok=True)
    for name in C.STANDARD:
        p, l = C.make_standard(name)
        C.save(os.path.join(OUT, name + ".txt"), p, l, f"{name}: conventional layout (oracle.constellation)")
        print(name, "written")
    p8, l8 = C.make_standard("QAM8")
    g0 = shaping.gmi_awgn(p8, l8, 14.0)
    p, l, tr = shaping.optimize(p8, l8, 14.0, iters=a.gs8_iters, seed=8)
    C.save(os.path.join(OUT, "GS8.txt"), p, l,
           f"GS-8: oracle.shaping.optimize(QAM8, 14 dB, iters={a.gs8_iters}, seed=8)\n"
           f"GMI(QAM8,14dB)={g0:.6f}  GMI(GS8,14dB)={tr[-1]:.6f}")
    print("GS8", g0, tr[-1])
    p128, l128 = C.make_standard("QAM128")
    g0 = shaping.gmi_awgn(p128, l128, 20.0, order=6)
    p, l, tr = shaping.optimize(p128, l128, 20.0, iters=a.gs128_iters, seed=128, sym4=True, order=6)
    C.save(os.path.join(OUT, "GS128.txt"), p, l,
           f"GS-128: oracle.shaping.optimize(QAM128, 20 dB, iters={a.gs128_iters}, seed=128, quadrant symmetry)\n"
           f"GMI(QAM128,20dB)={g0:.6f}  GMI(GS128,20dB)={tr[-1]:.6f}")
    print("GS128", g0, tr[-1])


if __name__ == "__main__":
    main()
