"""Small streaming workload for compute-sanitizer (racecheck / synccheck / memcheck).

Exercises every launch shape of the product path on 2^16-sample C2 buffers:
  * kk_rx_process_batch (tail launch, kk_lms_kernel, chain APPLY launch),
  * kk_rx_submit_batch / kk_rx_sync with 2-buffer batches (in-launch warp-per-chain
    update-pass CTAs spinning on the launch's tail-completion counter),
  * kk_rx_submit_batch with 64-buffer batches (the in-launch lane-per-chain CTA),
and checks that the streamed labels equal the synchronous ones (so a sanitizer run that
perturbs scheduling still has to produce the same result).

usage: python tools/sanitize_run.py [nbig] [labels.npy]   (under gpurun; compute-sanitizer or a KK_JITTER build)
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2108_07004_b200 import KKReceiver, halo_for  # noqa: E402
from synth import configs  # noqa: E402
from synth.generate import make_pool, make_stream  # noqa: E402

nbig = int(sys.argv[1]) if len(sys.argv) > 1 else 64
name = "C2_n16"
cfg = configs.get(name).link
pool = make_pool(cfg, 6)
h = np.loadtxt(os.path.join(ROOT, "data", "fir", name + ".txt"))
fir = h[:, 0] + 1j * h[:, 1]
left, right = halo_for(cfg.buffer_len)
nbuf = 4 + nbig
st, off = make_stream(pool, nbuf, left, right)
n_sym = cfg.buffer_len // 4
src = torch.from_numpy(st).cuda()


def rx():
    return KKReceiver(cfg.fmt, cfg.buffer_len, cfg.cspr_db, fir, pool.dc_offset, tone_bin=cfg.tbin,
                      ref_pattern=pool.pattern, max_batch=nbig)


ref = rx()
out_ref = torch.empty(nbuf * n_sym, dtype=torch.uint8, device="cuda")
ref.process_batch(src, off, 4, out_ref[: 4 * n_sym])
ref.process_batch(src, off + 4 * cfg.buffer_len, nbig, out_ref[4 * n_sym:])
torch.cuda.synchronize()

r = rx()
out = torch.empty(nbuf * n_sym, dtype=torch.uint8, device="cuda")
r.submit_batch(src, off, 2, out[: 2 * n_sym])
r.submit_batch(src, off + 2 * cfg.buffer_len, 2, out[2 * n_sym: 4 * n_sym])
r.submit_batch(src, off + 4 * cfg.buffer_len, nbig, out[4 * n_sym:])
r.sync()
torch.cuda.synchronize()
same = bool(torch.equal(out, out_ref))
print(f"sanitize_run: {nbuf} buffers, streamed == synchronous: {same}", flush=True)
if len(sys.argv) > 2:  # save the labels to compare builds (tools/gpu/race_jitter.sh)
    np.save(sys.argv[2], out.cpu().numpy())
r.close()
ref.close()
sys.exit(0 if same else 1)
