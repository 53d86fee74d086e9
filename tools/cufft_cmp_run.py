"""Run the cuFFT comparison pipeline (libkkrx_cufft.so) on B C5 buffers, for ncu.

    python tools/cufft_cmp_run.py [B] [reps]
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum ... python tools/cufft_cmp_run.py 16 2
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2108_07004_b200 import halo_for  # noqa: E402
from paper_2108_07004_b200.cufft_cmp import CufftS1S4  # noqa: E402
from synth import configs  # noqa: E402
from synth.generate import make_pool, make_stream  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 16
R = int(sys.argv[2]) if len(sys.argv) > 2 else 2
cfg = configs.get("C5").link
N = cfg.buffer_len
pool = make_pool(cfg, B)
h = np.loadtxt(os.path.join(ROOT, "data", "fir", "C5.txt"))
fir = h[:, 0] + 1j * h[:, 1]
left, right = halo_for(N)
stream, off = make_stream(pool, B, left, right)
d = torch.from_numpy(stream).cuda()
cm = CufftS1S4(N, B, pool.dc_offset, cfg.cspr_db, fir, tone_bin=cfg.tbin)
x2 = torch.empty(B * N // 2, dtype=torch.complex64, device="cuda")
for _ in range(R):
    cm.x2(d, off, B, x2)
torch.cuda.synchronize()
print("ok", B, R, float(x2.abs().mean()))
