"""Device timeline (CUPTI via torch.profiler) of one kk_rx_train_fir and one
kk_rx_train_taps call on a C5 buffer.  python tools/train_timeline.py"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2108_07004_b200 import KKReceiver, halo_for  # noqa: E402
from synth import configs  # noqa: E402
from synth.generate import make_pool, make_stream  # noqa: E402

cfg = configs.get("C5").link
N = cfg.buffer_len
left, right = halo_for(N)
tr = make_pool(cfg, 1, noiseless=True, cache=False)
st, off = make_stream(tr, 1, left, right)
src = torch.from_numpy(st).cuda()
sym = tr.points[tr.pattern.astype(np.int64)]
rx = KKReceiver("CUSTOM", N, cfg.cspr_db, np.zeros(203), tr.dc_offset, points=tr.points, labels=tr.labels,
                tone_bin=cfg.tbin, ref_pattern=tr.pattern)
rx.train_fir(src, off, sym[32:32 + 8192], 32)
for name, fn in (("train_fir", lambda: rx.train_fir(src, off, sym[32:32 + 8192], 32)),
                 ("train_taps", lambda: rx.train_taps(src, off, 4096))):
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        t0 = time.perf_counter()
        fn()
        wall = (time.perf_counter() - t0) * 1e3
    ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    ev.sort(key=lambda e: e.time_range.start)
    print(f"== {name}: wall {wall:.1f} ms")
    for e in ev:
        print(f"   {(e.time_range.end - e.time_range.start) / 1e3:9.3f} ms  {e.name[:70]}")
