"""Device timeline of the streaming pipeline (CUPTI via torch.profiler): every kernel,
memset and memcpy of a few kk_rx_submit_batch steps with start/duration/gap, to find
where the per-step time outside the chain launch goes.  python tools/pipeline_timeline.py [B] [steps]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import time  # noqa: E402
import numpy as np  # noqa: E402
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2108_07004_b200 import KKReceiver, halo_for  # noqa: E402
from synth import configs  # noqa: E402
from synth.generate import make_pool, make_stream  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
S = int(sys.argv[2]) if len(sys.argv) > 2 else 6
MODE = sys.argv[3] if len(sys.argv) > 3 and not sys.argv[3].startswith("-") else "dev"  # dev | int16 | packed
cfg = configs.get("C5").link
N = cfg.buffer_len
P = 16
pool = make_pool(cfg, P)
h = np.loadtxt(os.path.join(ROOT, "data", "fir", "C5.txt"))
fir = h[:, 0] + 1j * h[:, 1]
left, right = halo_for(N)
st, off = make_stream(pool, P + B, left, right)
if MODE == "dev":
    d = torch.from_numpy(st).cuda()
    out = [torch.empty(B * N // 4, dtype=torch.uint8, device="cuda") for _ in range(2)]
elif MODE == "packed":
    from synth.generate import pack12
    d = torch.from_numpy(pack12(st)).pin_memory()
    out = [torch.empty(B * N // 4, dtype=torch.uint8).pin_memory() for _ in range(2)]
else:
    d = torch.from_numpy(st).pin_memory()
    out = [torch.empty(B * N // 4, dtype=torch.uint8).pin_memory() for _ in range(2)]
submit = rx_submit = None
cur = torch.cuda.current_stream()
rx = KKReceiver("CUSTOM", N, cfg.cspr_db, fir, pool.dc_offset, points=pool.points, labels=pool.labels,
                tone_bin=cfg.tbin, ref_pattern=pool.pattern, stream=cur.cuda_stream, max_batch=B)
def sub(s, b0):
    if MODE == "packed":
        rx.submit_batch_packed12(d, off + b0 * N, B, out[s & 1])
    else:
        rx.submit_batch(d, off + b0 * N, B, out[s & 1])


for s in range(3):
    sub(s, (s * B) % P)
rx.sync()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for s in range(S):
        b0 = (s * B) % P
        rx.seek(b0)
        sub(s, b0)
    rx.sync()
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ev.sort(key=lambda e: e.time_range.start)
t0 = ev[0].time_range.start
prev_end = None
verbose = "-v" in sys.argv
tot_gap = 0.0
chain = []
for e in ev:
    s_, e_ = e.time_range.start, e.time_range.end
    gap = (s_ - prev_end) if prev_end is not None else 0
    tot_gap += max(gap, 0)
    if "chain" in e.name:
        chain.append(e_ - s_)
    if verbose or gap > 20:
        print(f"{(s_ - t0) / 1e3:9.3f} ms  dur {(e_ - s_) / 1e3:8.4f} ms  gap {gap / 1e3:7.4f} ms  {e.name[:60]}")
    prev_end = e_ if prev_end is None else max(prev_end, e_)
span = (prev_end - t0) / 1e3
print(f"span {span:.3f} ms for {S} steps = {span / S:.4f} ms/step; device gaps {tot_gap / 1e3:.3f} ms; "
      f"chain launches {len(chain)} avg {np.mean(chain) / 1e3:.4f} ms min {np.min(chain) / 1e3:.4f} max {np.max(chain) / 1e3:.4f}")
print("chain durations (ms):", " ".join(f"{c / 1e3:.3f}" for c in chain))

# the same loop timed with CUDA events and host wall clock, without the profiler
for rep in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter() if "time" in globals() else None
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(cur)
    for s in range(S):
        b0 = (s * B) % P
        rx.seek(b0)
        sub(s, b0)
    rx.sync()
    e1.record(cur)
    torch.cuda.synchronize()
    print(f"events: {e0.elapsed_time(e1) / S:.4f} ms/step")
