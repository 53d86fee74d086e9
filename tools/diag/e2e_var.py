"""Run-to-run spread of the end-to-end (pinned host input) rate: packed-12 and int16
submissions, several repetitions per batch size.  python tools/e2e_var.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2108_07004_b200 import KKReceiver, halo_for  # noqa: E402
from synth import configs  # noqa: E402
from synth.generate import make_pool, make_stream, pack12  # noqa: E402

cfg = configs.get("C5").link
N = cfg.buffer_len
P = 16
pool = make_pool(cfg, P)
h = np.loadtxt(os.path.join(ROOT, "data", "fir", "C5.txt"))
fir = h[:, 0] + 1j * h[:, 1]
left, right = halo_for(N)
cur = torch.cuda.current_stream()
for B in (64, 128):
    st, off = make_stream(pool, P + B, left, right)
    hp = torch.from_numpy(pack12(st)).pin_memory()
    hs = torch.from_numpy(st).pin_memory()
    out = [torch.empty(B * N // 4, dtype=torch.uint8).pin_memory() for _ in range(2)]
    rx = KKReceiver("CUSTOM", N, cfg.cspr_db, fir, pool.dc_offset, points=pool.points, labels=pool.labels,
                    tone_bin=cfg.tbin, ref_pattern=pool.pattern, stream=cur.cuda_stream, max_batch=B)
    res = {"packed": [], "int16": []}
    for rep in range(4):
        for kind in ("packed", "int16"):
            def sub(s):
                if kind == "packed":
                    rx.submit_batch_packed12(hp, off, B, out[s & 1])
                else:
                    rx.submit_batch(hs, off, B, out[s & 1])
            sub(0)
            rx.sync()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(cur)
            S = 10
            for s in range(S):
                sub(s)
            rx.sync()
            e1.record(cur)
            torch.cuda.synchronize()
            res[kind].append(round(S * B * N / (e0.elapsed_time(e1) / 1e3) / 1e9, 2))
    print(B, res, flush=True)
    rx.close()
    del hp, hs, out
