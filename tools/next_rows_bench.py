"""Measurements of the SURVEY 8(f) NEXT rows on the GPU (their parity is in
tests/test_gpu_parity.py; this is the measurement half of the bar).  C5 workload, full
2^22-sample buffers, device-resident, CUDA events on the receiver's stream.

    python tools/next_rows_bench.py [B] > profiles/.../next_rows.json

  row 1  DC-offset sweep (kk_rx_dc_sweep): 5 hypotheses over B buffers
  row 2  init-time training: kk_rx_frame_sync (all 2^20 lags), kk_rx_train_fir (LS 203
         taps from 8192 symbols) and kk_rx_train_taps (4096 PILOT LMS steps)
  row 3  pre-KK intensity equaliser: streaming throughput with a 15-tap pre-FIR vs without
  row 4  GMI of constellations (kk_gmi_awgn): batched evaluations per second
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2108_07004_b200 import KKReceiver, gmi_awgn, halo_for  # noqa: E402
from synth import configs  # noqa: E402
from synth.generate import load_constellation, make_pool, make_stream  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
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
kw = dict(points=pool.points, labels=pool.labels, tone_bin=cfg.tbin, ref_pattern=pool.pattern,
          stream=cur.cuda_stream, max_batch=B)


def timed(fn, reps=1):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(cur)
    for _ in range(reps):
        r = fn()
    e1.record(cur)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps, r


def stream_rate(rx, steps=10):
    def run():
        for s in range(steps):
            rx.submit_batch(d, off, B, out[s & 1])
        return rx.sync()
    run()
    ms, _ = timed(run)
    return steps * B * N / (ms / 1e3) / 1e9


res = {"workload": f"C5 (GS-128), 2^22-sample buffers, {B} per call, device-resident", "unit": "GSa/s"}
# row 3: pre-KK equaliser on vs off (tap values do not change the work; a unit-DC-gain 15-tap FIR)
g = np.zeros(15, np.float32)
g[7] = 0.8
g[6] = g[8] = 0.1
rx0 = KKReceiver("CUSTOM", N, cfg.cspr_db, fir, pool.dc_offset, **kw)
rx1 = KKReceiver("CUSTOM", N, cfg.cspr_db, fir, pool.dc_offset, pre_fir=g, **kw)
v0, v1 = stream_rate(rx0), stream_rate(rx1)
res["row3_pre_kk_equaliser"] = {"value_without": v0, "value_with_15_taps": v1, "ratio": v1 / v0,
                                "kernel": "kk_chain_kernel<PREKK=true> (FIR fused into the S1/S3 code reads)"}
rx1.close()
# row 1: DC-offset sweep, 5 hypotheses (each a full S1-S7 pass over the B buffers)
dcs = [pool.dc_offset * f for f in (0.96, 0.98, 1.0, 1.02, 1.04)]
rx0.dc_sweep(d, off, B, dcs)
ms, (cnts, best) = timed(lambda: rx0.dc_sweep(d, off, B, dcs))
res["row1_dc_sweep"] = {"hypotheses": len(dcs), "buffers": B, "ms": ms,
                        "value": len(dcs) * B * N / (ms / 1e3) / 1e9, "best_index": best,
                        "note": "GSa/s of hypothesis-samples (each hypothesis is a full S1-S7 pass)"}
rx0.close()
# row 2: init-time training
tr = make_pool(cfg, 1, noiseless=True, cache=False)
st_t, off_t = make_stream(tr, 1, left, right)
src_t = torch.from_numpy(st_t).cuda()
sym = tr.points[tr.pattern.astype(np.int64)]
rx2 = KKReceiver("CUSTOM", N, cfg.cspr_db, np.zeros(203), tr.dc_offset, points=tr.points, labels=tr.labels,
                 tone_bin=cfg.tbin, ref_pattern=tr.pattern, stream=cur.cuda_stream)
def wall(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) * 1e3 / reps


t_fir = wall(lambda: rx2.train_fir(src_t, off_t, sym[32:32 + 8192], 32))
rx2.set_fir(fir)
t_taps = wall(lambda: rx2.train_taps(src_t, off_t, 4096))
t_fs = wall(lambda: rx2.frame_sync(src_t, off_t, 64, 2048))
fs = rx2.frame_sync(src_t, off_t, 64, 2048)
res["row2_training"] = {"train_fir_ms": t_fir, "train_fir": "LS 203-tap FIR from 8192 training symbols (fp64 Gram + Cholesky on the GPU), host wall time incl. the copy-back",
                        "train_taps_ms": t_taps, "train_taps": "4096 PILOT LMS steps from W_init, host wall time",
                        "frame_sync_ms": t_fs, "frame_sync": "all 2^20 cyclic lags x 2048 symbol-instant samples "
                        "(E_s of one buffer + kk_fsync_kernel), host wall time",
                        "frame_sync_result": {"n_off": fs[0], "peak_to_mean": fs[2]}}
rx2.close()
# row 4: GMI evaluations per second (GS-128 at 20 dB, Gauss-Hermite order 6, batches of 256 label permutations)
pts, labs = load_constellation("GS128")
rng = np.random.default_rng(1)
P4 = np.stack([pts] * 256)
L4 = np.stack([rng.permutation(labs) for _ in range(256)])
gmi_awgn(P4, L4, 20.0, 6)
t0 = time.perf_counter()
for _ in range(5):
    gmi_awgn(P4, L4, 20.0, 6)
dt = (time.perf_counter() - t0) / 5
res["row4_gmi"] = {"evaluations_per_s": 256 / dt, "batch": 256, "constellation": "GS-128", "order": 6}
print(json.dumps(res, indent=1))
