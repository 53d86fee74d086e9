"""Write data/fir/<workload>.txt: the 203-tap static-EQ input for each workload.

PAPER l.53: the static equaliser "is optimized offline using a training sequence
every time that the data acquisition is initialized".  Here: the LS fit of
oracle.train.train_fir on the noiseless training buffer of the workload (same
signal, same ADC gain; synth.generate.make_pool(noiseless=True)) over the first
TRAIN_SYMS symbols.  The taps are an INPUT of kk_rx_create / oracle.receive, so
both sides read the same committed file.  Only oracle/ (arithmetic) and synth/
(input generation) are called.

Run:  python tools/make_fixtures.py [name-regex]
"""
import os
import re
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import kk_oracle as O  # noqa: E402
from oracle import train  # noqa: E402
from synth import configs  # noqa: E402
from synth.generate import make_pool, make_stream  # noqa: E402

TRAIN_SYMS = 16384
FIR_DIR = os.path.join(ROOT, "data", "fir")


def fit_for(wl):
    cfg = wl.link
    pool = make_pool(cfg, 1, cache=False, noiseless=True)
    margin = 2048
    st, off = make_stream(pool, 1, margin, margin)
    win = st[:off + 4 * TRAIN_SYMS + margin]
    p = O.RxParams(buffer_len=cfg.buffer_len, cspr_db=cfg.cspr_db, dc_offset=pool.dc_offset,
                   fir=np.zeros(O.FIR_TAPS), points=pool.points, labels=pool.labels, tone_bin=cfg.tbin)
    sym = pool.points[pool.pattern.astype(np.int64)]
    return train.train_fir(win, off, p, sym[:TRAIN_SYMS], 0, TRAIN_SYMS)


def write_fir(path, h, name):
    with open(path, "w") as f:
        f.write(f"# 203-tap static EQ for workload {name}: LS fit (oracle.train.train_fir) on the\n")
        f.write(f"# noiseless training buffer, {TRAIN_SYMS} symbols. Tap i = line - 101. Columns: re im\n")
        for v in h:
            f.write(f"{v.real:+.17e} {v.imag:+.17e}\n")


def main():
    pat = re.compile(sys.argv[1]) if len(sys.argv) > 1 else None
    os.makedirs(FIR_DIR, exist_ok=True)
    for name, wl in sorted(configs.ALL.items()):
        if pat and not pat.search(name):
            continue
        h = fit_for(wl)
        write_fir(os.path.join(FIR_DIR, name + ".txt"), h, name)
        print(name, "peak tap", int(np.argmax(np.abs(h))) - 101, "|h|max", float(np.abs(h).max()), flush=True)


if __name__ == "__main__":
    main()
