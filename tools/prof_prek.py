"""Small fixed workload for an ncu capture of the pre-KK instantiation (kk_chain_kernel<true>):
C5 buffers (pool of 4 cycled), device-resident, 32 buffers per call, a unit-DC-gain 15-tap
pre-FIR; 3 process_batch calls.  usage: python tools/prof_prek.py [nbuf]"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2108_07004_b200 import KKReceiver, halo_for  # noqa: E402
from synth import configs  # noqa: E402
from synth.generate import make_pool, make_stream  # noqa: E402

nb = int(sys.argv[1]) if len(sys.argv) > 1 else 32
cfg = configs.get("C5").link
pool = make_pool(cfg, 4)
h = np.loadtxt(os.path.join(ROOT, "data", "fir", "C5.txt"))
fir = h[:, 0] + 1j * h[:, 1]
g = np.zeros(15, np.float32)
g[7], g[6], g[8] = 0.8, 0.1, 0.1
left, right = halo_for(cfg.buffer_len)
st, off = make_stream(pool, nb, left, right)
d = torch.from_numpy(st).cuda()
out = torch.empty(nb * cfg.buffer_len // 4, dtype=torch.uint8, device="cuda")
rx = KKReceiver("CUSTOM", cfg.buffer_len, cfg.cspr_db, fir, pool.dc_offset, points=pool.points, labels=pool.labels,
                tone_bin=cfg.tbin, ref_pattern=pool.pattern, max_batch=nb, pre_fir=g)
for _ in range(3):
    c = rx.process_batch(d, off, nb, out)
torch.cuda.synchronize()
print("ok", c[0]["bit_errors"])
