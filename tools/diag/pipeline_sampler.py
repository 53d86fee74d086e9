"""Does the nvidia-smi clock sampler (bench.py ClockSampler) perturb the timed region?
Times the 30-step kk_rx_submit_batch loop with CUDA events, alternately without and with
the sampler.  python tools/pipeline_sampler.py"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2108_07004_b200 import KKReceiver, halo_for  # noqa: E402
from synth import configs  # noqa: E402
from synth.generate import make_pool, make_stream  # noqa: E402

B, S = 64, 30
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


def loop():
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    w0 = time.perf_counter()
    e0.record(cur)
    for s in range(S):
        rx.seek(0)
        rx.submit_batch(d, off, B, out[s & 1])
    rx.sync()
    e1.record(cur)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / S, (time.perf_counter() - w0) * 1e3 / S


for s in range(3):
    rx.submit_batch(d, off, B, out[s & 1])
rx.sync()
for rep in range(3):
    a = loop()
    with bench.ClockSampler(0) as clk:
        b = loop()
    print(f"no sampler: {a[0]:.4f} ms/step (wall {a[1]:.4f})   sampler: {b[0]:.4f} ms/step (wall {b[1]:.4f})  "
          f"clocks {clk.summary()}")
