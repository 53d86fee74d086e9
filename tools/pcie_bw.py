"""PCIe ceiling for bench.py's e2e number: pinned host<->device copy bandwidth on this box.

Times (CUDA events) the e2e leg's per-step transfer sizes -- the packed 12-bit H2D span
(805 MB for C5 at 128 buffers) and the symbol/count D2H (134 MB) -- alone and
concurrently on two streams, so e2e GSa/s can be read against the copy ceiling:
    e2e ceiling GSa/s = samples per step / max(H2D time, D2H time when overlapped).

    python tools/pcie_bw.py [B=128] > profiles/.../pcie_bw.json
"""
import json
import sys

import torch

B = int(sys.argv[1]) if len(sys.argv) > 1 else 128
N = 1 << 22
h2d_bytes = (B * N + 2 * 4096) * 3 // 2
d2h_bytes = B * (N // 4) + B * 64
dev = torch.device("cuda:0")
hs = torch.empty(h2d_bytes, dtype=torch.uint8).pin_memory()
ho = torch.empty(d2h_bytes, dtype=torch.uint8).pin_memory()
ds = torch.empty(h2d_bytes, dtype=torch.uint8, device=dev)
do = torch.zeros(d2h_bytes, dtype=torch.uint8, device=dev)
s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def h2d():
    ds.copy_(hs, non_blocking=True)


def d2h():
    ho.copy_(do, non_blocking=True)


def both():
    cur = torch.cuda.current_stream()
    ev = torch.cuda.Event()
    ev.record(cur)
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        ds.copy_(hs, non_blocking=True)
    with torch.cuda.stream(s2):
        ho.copy_(do, non_blocking=True)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


t_h = timed(h2d)
t_d = timed(d2h)
t_b = timed(both)
samples = B * N
res = {"buffers_per_step": B, "h2d_bytes": h2d_bytes, "d2h_bytes": d2h_bytes,
       "h2d_ms": t_h, "h2d_gbs": h2d_bytes / t_h / 1e6,
       "d2h_ms": t_d, "d2h_gbs": d2h_bytes / t_d / 1e6,
       "both_concurrent_ms": t_b,
       "e2e_ceiling_gsa": samples / t_b / 1e6,
       "e2e_ceiling_note": "samples per step / (H2D + D2H of one step on two streams); the pinned-copy bound of bench.py's e2e leg"}
print(json.dumps(res, indent=1))
