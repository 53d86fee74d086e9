"""Small fixed workload for ncu captures: 4 full-size (2^22) buffers of C1-shaped
data (pool of 1 cycled), device-resident, max_batch 4; 3 process_batch calls."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2108_07004_b200 import KKReceiver, halo_for  # noqa: E402
from synth import configs  # noqa: E402
from synth.generate import make_pool, make_stream  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C5"
nb = int(sys.argv[2]) if len(sys.argv) > 2 else 4
wl = configs.get(name)
cfg = wl.link
pool = make_pool(cfg, 1)
h = np.loadtxt(os.path.join(ROOT, "data", "fir", name + ".txt"))
fir = h[:, 0] + 1j * h[:, 1]
left, right = halo_for(cfg.buffer_len)
st, off = make_stream(pool, nb, left, right)
d = torch.from_numpy(st).cuda()
out = torch.empty(nb * cfg.buffer_len // 4, dtype=torch.uint8, device="cuda")
rx = KKReceiver("CUSTOM", cfg.buffer_len, cfg.cspr_db, fir, pool.dc_offset, points=pool.points, labels=pool.labels,
                tone_bin=cfg.tbin, ref_pattern=pool.pattern, max_batch=nb)
rx.set_timing(True)
for _ in range(3):
    c = rx.process_batch(d, off, nb, out)
torch.cuda.synchronize()
print({k: (v[0] / max(v[1], 1)) for k, v in rx.kernel_times().items()}, c[0])
