"""Write data/fir/<workload>.txt: the 203-tap static-EQ input for each workload.

PAPER l.53: the static equaliser "is optimized offline using a training sequence
every time that the data acquisition is initialized" -- i.e. on the live link, noise
included.  Here (reading R4): the least-squares fit of
oracle.train.train_fir over TRAIN_SYMS known symbols of a NOISY training stream of the
workload's link (same signal, ADC gain, OSNR and noise mode; a held-out noise seed,
seed_noise + TRAIN_SEED_OFFSET, so no buffer the tests or the bench receive is trained
on), made unbiased (h / g, g = the fit's gain on the training symbols).  On noisy data
the LS fit is the sample MMSE filter, which also rejects the out-of-band noise the KK
front end folds in (a fit on the noiseless twin leaves the stopband free and passed
~1.7 dB of extra noise on the two-sided configs, round-1 VERDICT).  Noiseless
workloads (C1) train on their noiseless buffer.

The taps are an INPUT of kk_rx_create / oracle.receive, so both sides read the same
committed file.  Only oracle/ (arithmetic) and synth/ (input generation) are called.

Run:  python tools/make_fixtures.py [name-regex]
"""
import os
import re
import sys
from dataclasses import replace
from multiprocessing import Pool as MPPool

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import kk_oracle as O  # noqa: E402
from oracle import train  # noqa: E402
from synth import configs  # noqa: E402
from synth.generate import make_pool, make_stream  # noqa: E402

TRAIN_SYMS = 65536
TRAIN_SEED_OFFSET = 7919
RIDGE = float(os.environ.get("FIXTURE_RIDGE", "1e-4"))
FIR_DIR = os.path.join(ROOT, "data", "fir")


def training_link(cfg):
    """The link the static EQ is trained on: the workload's link with a held-out noise seed."""
    return replace(cfg, seed_noise=cfg.seed_noise + TRAIN_SEED_OFFSET)


def fit_for(wl):
    cfg = wl.link
    nb = -(-TRAIN_SYMS // cfg.n_sym)
    if cfg.osnr_db is None:
        pool = make_pool(cfg, 1, cache=False, noiseless=True)
    else:
        pool = make_pool(training_link(cfg), nb, cache=False)
    margin = 2048
    st, off = make_stream(pool, nb, margin, margin)
    p = O.RxParams(buffer_len=cfg.buffer_len, cspr_db=cfg.cspr_db, dc_offset=pool.dc_offset,
                   fir=np.zeros(O.FIR_TAPS), points=pool.points, labels=pool.labels, tone_bin=cfg.tbin)
    sym = np.tile(pool.points[pool.pattern.astype(np.int64)], nb)[:TRAIN_SYMS]
    win = st[:off + 4 * TRAIN_SYMS + margin]
    return train.train_fir(win, off, p, sym, 0, TRAIN_SYMS, ridge=RIDGE, unbiased=True)


def write_fir(path, h, name, noiseless):
    src = "noiseless training buffer" if noiseless else \
        f"noisy training stream (noise seed + {TRAIN_SEED_OFFSET})"
    with open(path, "w") as f:
        f.write(f"# 203-tap static EQ for workload {name}: unbiased LS/MMSE fit (oracle.train.train_fir) on the\n")
        f.write(f"# {src}, {TRAIN_SYMS} symbols. Tap i = line - 101. Columns: re im\n")
        for v in h:
            f.write(f"{v.real:+.17e} {v.imag:+.17e}\n")


def _one(name):
    wl = configs.ALL[name]
    h = fit_for(wl)
    write_fir(os.path.join(FIR_DIR, name + ".txt"), h, name, wl.link.osnr_db is None)
    return name, int(np.argmax(np.abs(h))) - 101, float(np.abs(h).max())


def main():
    pat = re.compile(sys.argv[1]) if len(sys.argv) > 1 else None
    os.makedirs(FIR_DIR, exist_ok=True)
    names = [n for n in sorted(configs.ALL) if not pat or pat.search(n)]
    procs = int(os.environ.get("FIXTURE_PROCS", "4"))
    with MPPool(procs) as mp:
        for name, peak, hmax in mp.imap_unordered(_one, names):
            print(name, "peak tap", peak, "|h|max", hmax, flush=True)


if __name__ == "__main__":
    main()
