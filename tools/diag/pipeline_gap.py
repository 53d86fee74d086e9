"""Streaming-pipeline overhead per step: kk_rx_submit_batch loop with per-kernel timing on
and off, vs the chain-launch time.  python tools/pipeline_gap.py [B] [steps]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2108_07004_b200 import KKReceiver, halo_for  # noqa: E402
from synth import configs  # noqa: E402
from synth.generate import make_pool, make_stream  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
S = int(sys.argv[2]) if len(sys.argv) > 2 else 20
cfg = configs.get("C5").link
N = cfg.buffer_len
P = 16
pool = make_pool(cfg, P)
h = np.loadtxt(os.path.join(ROOT, "data", "fir", "C5.txt"))
fir = h[:, 0] + 1j * h[:, 1]
left, right = halo_for(N)
st, off = make_stream(pool, P + B, left, right)
d = torch.from_numpy(st).cuda()
out = [torch.empty(B * N // 4, dtype=torch.uint8, device="cuda") for _ in range(2)]
cur = torch.cuda.current_stream()
rx = KKReceiver("CUSTOM", N, cfg.cspr_db, fir, pool.dc_offset, points=pool.points, labels=pool.labels,
                tone_bin=cfg.tbin, ref_pattern=pool.pattern, stream=cur.cuda_stream, max_batch=B)


def run(timing):
    for s in range(3):
        rx.seek((s * B) % P)
        rx.submit_batch(d, off + ((s * B) % P) * N, B, out[s & 1])
    rx.sync()
    torch.cuda.synchronize()
    rx.set_timing(timing)
    rx.kernel_times()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(cur)
    for s in range(S):
        b0 = (s * B) % P
        rx.seek(b0)
        rx.submit_batch(d, off + b0 * N, B, out[s & 1])
    rx.sync()
    e1.record(cur)
    torch.cuda.synchronize()
    kt = rx.kernel_times()
    rx.set_timing(False)
    return e0.elapsed_time(e1) / S, kt


for timing in (False, True, False, True):
    ms, kt = run(timing)
    print(f"timing={timing}: {ms:.4f} ms/step  {B * N / ms / 1e6:.2f} GSa/s  kernel_times={kt}")
