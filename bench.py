"""Throughput benchmark of the B200 KK receiver hot path (BASELINE.json metric).

A step = one pass of the whole hot path (S1..S7: front end, Hilbert, reconstruct,
static EQ + 4->2, LMS update pass, WL apply, decision, demap, count) over one
batch of `--batch` 2^22-sample buffers of the C5 workload (GS-128, CSPR 16 dB,
two-sided ASE at OSNR 35 dB) per GPU.  Inputs are resident in
HBM (`value`); `e2e` repeats the measurement through the same C-ABI call with
pinned HOST buffers (H2D of the batch + halos and D2H of the labels inside the
timed region).

  python bench.py [--gpus N --steps K --warmup W]            # this implementation
  python bench.py --impl reference [--steps K --warmup W]    # the float64 CPU oracle
  torchrun --nproc-per-node N bench.py --gpus N ...          # one rank per GPU (weak scaling)

Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import math
import multiprocessing as mp
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "sustained GSa/s (equiv. GBaud) on full KK chain, 1/2/4/8 B200; % HBM roofline"
UNIT = "GSa/s"
# algorithmic work per ADC sample
HBM_BYTES_PER_SA = 2.25          # int16 in + uint8 label per 4 samples out
FLOP_PER_SA_KERNEL = 238.0       # kk_chain_kernel<APPLY>: Hilbert 100 + static EQ 97 + pointwise S1/S3 20
                                 # + WL apply 16 + decision ~5 (everything but the update pass)
FLOP_PER_SA_CHAIN = 240.0        # whole chain (+ WL apply 16, decision ~5, update ~0.2)
# FP32 SIMT peak derived from the unit counts and max clock (B200_PROFILING.md):
# 148 SMs x 128 FP32 lanes x 2 flop (FFMA) x 1.965 GHz
FP32_PEAK_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12
FP32_MEASURED_TFLOPS = 7.652 * 32 * 2 * 148 / 1e3  # tools/microbench/f32x2_rate.cu, 32 warps/SM


def cpu_model():
    """The host CPU model (lscpu "Model name"), stated beside the cpu_baseline core count."""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.lower().startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def _env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


class ClockSampler:
    """nvidia-smi clocks / throttle reasons streamed every 20 ms during the timed region
    (B200_PROFILING.md "clocks DURING the timed region")."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "20"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            time.sleep(0.3)  # let the first samples arrive before the timed region starts
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is None:
            return
        time.sleep(0.05)
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out, _ = self.proc.communicate()
        for line in (out or "").splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) >= 7:
                self.samples.append(f)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}

        def num(x):
            try:
                return float(x)
            except ValueError:
                return None
        sm = [num(s[0]) for s in self.samples if num(s[0]) is not None]
        smax = [num(s[1]) for s in self.samples if num(s[1]) is not None]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for s in self.samples:
            for n, v in zip(names, s[3:7]):
                if v.strip().lower() in ("active", "1"):
                    reasons.add(n)
        # only the samples taken under load (the sampler starts 0.3 s before the timed region)
        load = sorted(sm)[len(sm) // 4:] if len(sm) > 4 else sm
        return {"sm_mhz": statistics.median(load) if load else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(self.samples)}


def load_fir(name):
    h = np.loadtxt(os.path.join(ROOT, "data", "fir", f"{name}.txt"))
    return h[:, 0] + 1j * h[:, 1]


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {}


def issue_limit(traffic, samples, launch_ms):
    """The chain kernel against the SM issue rate (148 SMs x 4 schedulers x 1.965 GHz warp
    instructions/s) with the warp-instruction count of the committed ncu capture
    (DESIGN.md "Issue limit")."""
    if not traffic or "chain_warp_inst_per_launch" not in traffic:
        return None
    ipsa = traffic["chain_warp_inst_per_launch"] / traffic["chain_samples_per_launch"]
    peak = 148 * 4 * 1.965e9
    bound = peak / ipsa / 1e9
    achieved = samples / (launch_ms / 1e3) / 1e9
    return {"warp_inst_per_sa": ipsa, "issue_bound_gsa": bound, "chain_gsa": achieved, "frac": achieved / bound,
            "source": traffic.get("inst_source")}


def profile_traffic():
    """dram bytes per kk_x2 launch from the committed `ncu --set full` capture."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            return json.load(f)
    except Exception:
        return None


# ----------------------------------------------------------------------------
# oracle (CPU) legs: cpu_baseline and --impl reference
# ----------------------------------------------------------------------------
def _oracle_one(args):
    name, b, n_pool = args
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    from oracle import kk_oracle as O
    from synth import configs
    from synth.generate import make_pool, make_stream
    wl = configs.get(name)
    cfg = wl.link
    pool = make_pool(cfg, n_pool)
    left, right = O.required_left(4096), 2304
    st, off = make_stream(pool, 1, left, right, first=b)
    p = O.RxParams(buffer_len=cfg.buffer_len, cspr_db=cfg.cspr_db, dc_offset=pool.dc_offset, fir=load_fir(name),
                   points=pool.points, labels=pool.labels, tone_bin=cfg.tbin, pattern=pool.pattern)
    t0 = time.perf_counter()
    r = O.receive(st, off, p)
    return time.perf_counter() - t0, r["bit_errors"], cfg.buffer_len


def oracle_rate(name, n_pool, workers, tasks):
    """Run `tasks` whole buffers through the oracle with `workers` processes.
    Returns (GSa/s, seconds, samples)."""
    ctx = mp.get_context("spawn")
    t0 = time.perf_counter()
    with ctx.Pool(workers) as pool:
        res = pool.map(_oracle_one, [(name, b % n_pool, n_pool) for b in range(tasks)])
    dt = time.perf_counter() - t0
    samples = sum(r[2] for r in res)
    return samples / dt / 1e9, dt, samples


def run_reference(args):
    """The reference arm: the float64 oracle (oracle/, as it stands) on the host cores, same
    workload / metric / unit.  A step is ONE whole C5 buffer (a bounded sample of the
    workload); the K steps run concurrently on `workers` host processes (spawn and input
    loading inside the timed region), so value = K buffers x 2^22 samples / wall time and the
    run ends within a minute or two whatever K is.  Under torchrun only rank 0 runs."""
    rank = _env_int("RANK", 0)
    if rank != 0:
        return 0
    workers = args.ref_workers or (os.cpu_count() or 1)
    from synth import configs
    from synth.generate import make_pool
    make_pool(configs.get(args.workload).link, args.pool)  # warm the input cache outside the timed steps
    oracle_rate(args.workload, args.pool, workers, min(max(args.warmup, 1), workers))  # W untimed buffers
    value, total, samples = oracle_rate(args.workload, args.pool, workers, args.steps)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": args.workload + " (GS-128 CSPR 16 dB two-sided OSNR 35 dB, 2^22-sample buffers)",
                   "buffers_per_step": 1, "host_processes": workers,
                   "l2": "inputs > L2 not applicable (CPU)"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": workers, "kind": "oracle", "cpu_model": cpu_model(),
                         "sample": f"{args.steps} whole 2^22-sample buffers (one per step) on {workers} processes "
                                   f"({total:.1f} s)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------
# GPU leg
# ----------------------------------------------------------------------------
def run_gpu(args):
    import torch
    import torch.distributed as dist

    world = _env_int("WORLD_SIZE", 1)
    rank = _env_int("RANK", 0)
    local = _env_int("LOCAL_RANK", 0)
    torch.cuda.set_device(local)
    # launched by torchrun (any world size, including 1): one NCCL process group, so the
    # multi-rank code path (barriers, the counter all_reduce, max-over-ranks timing) runs
    dist_on = world > 1 or "TORCHELASTIC_RUN_ID" in os.environ
    if dist_on:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        print(f"[bench] rank {rank}/{world} local {local}: process group backend {dist.get_backend()}, "
              f"world {dist.get_world_size()}", file=sys.stderr, flush=True)
    dev = torch.device("cuda", local)

    from paper_2108_07004_b200 import KKReceiver, halo_for
    from synth import configs
    from synth.generate import make_pool, make_stream

    from paper_2108_07004_b200.sharding import comm_info, max_over_ranks, rank_batches, reduce_counts, shard_range, \
        sum_counts

    wl = configs.get(args.workload)
    cfg = wl.link
    N = cfg.buffer_len
    B = args.batch
    P = args.pool
    S = args.stream or wl.n_buffers  # C5: the continuous 4096-buffer stream, sharded contiguously over the ranks
    # rank 0 generates (and caches) the pool first, then the others load it
    if rank == 0:
        pool = make_pool(cfg, P)
    if dist_on:
        dist.barrier()
    if rank != 0:
        pool = make_pool(cfg, P)
    fir = load_fir(args.workload)
    left, right = halo_for(N)
    # device-resident stream: pool cycled so every step's B buffers + halos are contiguous
    span = P + B
    stream_np, off = make_stream(pool, span, left, right, first=0)
    d_stream = torch.from_numpy(stream_np).to(dev)
    d_out = [torch.empty(B * (N // 4), dtype=torch.uint8, device=dev) for _ in range(3)]
    cur = torch.cuda.current_stream(dev)
    rx = KKReceiver("CUSTOM" if not cfg.fmt.startswith("QAM") else cfg.fmt, N, cfg.cspr_db, fir, pool.dc_offset,
                    points=pool.points, labels=pool.labels, tone_bin=cfg.tbin, ref_pattern=pool.pattern,
                    device=local, stream=cur.cuda_stream, max_batch=B)

    def batches(step):
        # this rank's batches of stream buffers in `step`: the S-buffer stream is sharded into
        # contiguous per-rank ranges (sharding.rank_batches; stream buffer b = pool buffer b % P,
        # whose window starts at off + (b % P) N in the cycled device layout)
        return rank_batches(step, rank, world, B, S, args.scaling)

    nsub = [0]

    # the streaming receiver: kk_rx_submit_batch per batch (the LMS update pass of batch
    # j overlaps the fused chain of batch j-1), kk_rx_sync once after the last step
    def submit_dev(s):
        for b0, cnt in batches(s):
            rx.seek(b0)
            rx.submit_batch(d_stream, off + (b0 % P) * N, cnt, d_out[nsub[0] % 3][: cnt * (N // 4)])
            nsub[0] += 1

    for s in range(args.warmup):
        submit_dev(s)
    rx.sync()
    torch.cuda.synchronize(dev)
    rx.set_timing(True)
    rx.async_launches()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    if dist_on:
        dist.barrier()
    torch.cuda.synchronize(dev)
    with ClockSampler(local) as clk:
        t0.record(cur)
        for s in range(args.steps):
            submit_dev(args.warmup + s)
        counts = rx.sync(as_array=True)  # counters as one array: no per-buffer Python objects in the timed region
        t1.record(cur)
        torch.cuda.synchronize(dev)
    if dist_on:
        dist.barrier()
    ms = t0.elapsed_time(t1)
    local = sum_counts(counts)
    launches = rx.async_launches()
    ktimes = rx.kernel_times()
    rx.set_timing(False)

    # the same steps through the synchronous call (one batch at a time, LMS pass not hidden)
    def step_sync(s):
        for b0, cnt in batches(s):
            rx.seek(b0)
            rx.process_batch(d_stream, off + (b0 % P) * N, cnt, d_out[0][: cnt * (N // 4)], as_array=True)
    step_sync(0)
    torch.cuda.synchronize(dev)
    s0 = torch.cuda.Event(enable_timing=True)
    s1 = torch.cuda.Event(enable_timing=True)
    s0.record(cur)
    for s in range(args.steps):
        step_sync(s)
    s1.record(cur)
    torch.cuda.synchronize(dev)
    sync_ms = max_over_ranks(s0.elapsed_time(s1), device=dev)
    # S8: the only data-path collective -- all_reduce(SUM) of the error counters, MAX of the time
    tot, ms_max = reduce_counts(local, ms, device=dev)
    samples_total = tot["symbols"] * 4  # every buffer the ranks processed in the timed steps (4 sps)
    value = samples_total / (ms_max / 1e3) / 1e9

    # ---------------- cuFFT comparison (north star: "cuFFT reported only as a comparison";
    # SURVEY 8(d)): S1-S4 of the same batches as a multi-kernel pipeline around cuFFT with
    # every intermediate in HBM (libkkrx_cufft.so).  It stops at x2; the fused chain above
    # also runs S5-S7.  Rank 0 at N = 1 only.
    cufft_cmp = None
    if world == 1 and not args.no_cufft:
        from paper_2108_07004_b200.cufft_cmp import CufftS1S4
        cm = CufftS1S4(N, B, pool.dc_offset, cfg.cspr_db, fir, tone_bin=cfg.tbin)
        x2_out = torch.empty(B * (N // 2), dtype=torch.complex64, device=dev)
        cm_first = [batches(s)[0][0] % P for s in range(max(args.warmup, args.steps))]
        for s in range(args.warmup):
            cm.x2(d_stream, off + cm_first[s] * N, B, x2_out, cur.cuda_stream)
        torch.cuda.synchronize(dev)
        c0 = torch.cuda.Event(enable_timing=True)
        c1 = torch.cuda.Event(enable_timing=True)
        c0.record(cur)
        for s in range(args.steps):
            cm.x2(d_stream, off + cm_first[s] * N, B, x2_out, cur.cuda_stream)
        c1.record(cur)
        torch.cuda.synchronize(dev)
        cms = c0.elapsed_time(c1)
        cv = args.steps * B * N / (cms / 1e3) / 1e9
        cufft_cmp = {"value": cv, "unit": UNIT, "ms_per_step": cms / args.steps, "stages": "S1-S4 (to x2)",
                     "launches_per_step": cm.launches(B),
                     "design": "pack -> cuFFT C2C 1024 -> mask -> cuFFT C2C 1024 -> S3 (E_s to HBM) -> cuFFT C2C "
                               "1024 over overlapping windows -> x H + fold -> cuFFT C2C 512 -> extract",
                     "fused_full_chain_over_cufft_s1_s4": value / cv}
        del x2_out
        cm.close()

    # ---------------- e2e through the same C-ABI with pinned host buffers
    e2e = None
    if not args.no_e2e:
        # the ADC's native packed 12-bit samples (1.5 B per sample) in pinned host memory, and
        # the int16 form of the same codes (2 B per sample) for comparison
        from synth.generate import pack12
        h_packed = torch.from_numpy(pack12(stream_np)).pin_memory()
        h_stream = torch.from_numpy(stream_np).pin_memory()
        h_out = [torch.empty(B * (N // 4), dtype=torch.uint8).pin_memory() for _ in range(3)]

        def submit_host(s, packed):
            for b0, cnt in batches(s):
                rx.seek(b0)
                o = h_out[nsub[0] % 3][: cnt * (N // 4)]
                nsub[0] += 1
                if packed:
                    rx.submit_batch_packed12(h_packed, off + (b0 % P) * N, cnt, o)
                else:
                    rx.submit_batch(h_stream, off + (b0 % P) * N, cnt, o)

        def e2e_run(packed):
            for s in range(args.warmup):  # W untimed steps (every pipeline slot and its staging)
                submit_host(s, packed)
            rx.sync(as_array=True)
            torch.cuda.synchronize(dev)
            if dist_on:
                dist.barrier()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(cur)
            for s in range(args.steps):
                submit_host(s, packed)
            rx.sync(as_array=True)
            e1.record(cur)
            torch.cuda.synchronize(dev)
            return samples_total / (max_over_ranks(e0.elapsed_time(e1), device=dev) / 1e3) / 1e9

        v_packed = e2e_run(True)
        v_int16 = e2e_run(False)
        span = left + B * N + right
        d2h = B * (N // 4) + B * 64

        # the PCIe ceiling of this leg on this box: one step's packed H2D and symbol D2H as
        # plain pinned copies on two streams (no kernels), CUDA events, 5 repetitions
        h_step = h_packed[:span * 3 // 2]
        d_scr = torch.empty(h_step.numel(), dtype=torch.uint8, device=dev)
        d_o = torch.zeros(h_out[0].numel(), dtype=torch.uint8, device=dev)
        cs1, cs2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)

        def copies():
            cs1.wait_stream(cur)
            cs2.wait_stream(cur)
            with torch.cuda.stream(cs1):
                d_scr.copy_(h_step, non_blocking=True)
            with torch.cuda.stream(cs2):
                h_out[0].copy_(d_o, non_blocking=True)
            cur.wait_stream(cs1)
            cur.wait_stream(cs2)

        copies()
        torch.cuda.synchronize(dev)
        p0 = torch.cuda.Event(enable_timing=True)
        p1 = torch.cuda.Event(enable_timing=True)
        p0.record(cur)
        for _ in range(5):
            copies()
        p1.record(cur)
        torch.cuda.synchronize(dev)
        pcie_ms = p0.elapsed_time(p1) / 5
        del d_scr, d_o
        e2e = {"value": v_packed, "unit": UNIT, "h2d_bytes_per_step": span * 3 // 2, "d2h_bytes_per_step": d2h,
               "input": "packed 12-bit ADC samples (kk_rx_submit_batch_packed12), pinned host memory",
               "int16_input_value": v_int16, "int16_h2d_bytes_per_step": span * 2,
               "pcie_ceiling": {"value": B * N / (pcie_ms / 1e3) / 1e9 * world, "unit": UNIT,
                                "ms_per_step": pcie_ms, "frac": v_packed / (B * N / (pcie_ms / 1e3) / 1e9 * world),
                                "basis": "one step's packed H2D + symbol D2H as plain pinned copies on two "
                                         "streams, no kernels (tools/pcie_bw.py)"}}

    if rank != 0:
        rx.close()
        if dist_on:
            dist.destroy_process_group()
        return 0

    peaks = measured_peaks()
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    ch_ms, ch_n = ktimes["chain"]
    if ch_n == 0:
        raise RuntimeError("no chain kernel timing recorded")
    ch_avg_ms = ch_ms / max(ch_n, 1)
    achieved_tf = FLOP_PER_SA_KERNEL * B * N / (ch_avg_ms / 1e3) / 1e12
    traffic = profile_traffic()
    step_ms = ms_max / args.steps
    lms_avg = ktimes["lms"][0] / max(ktimes["lms"][1], 1)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True, "scaling": args.scaling,
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"{args.workload}: GS-128, CSPR 16 dB, two-sided ASE at OSNR 35 dB, "
                               f"2^22-sample 12-bit buffers; a continuous {S}-buffer stream (pool of {P} distinct "
                               f"buffers cycled) sharded contiguously over {world} GPU(s); "
                               + (f"{B} buffers/step/GPU walking each rank's own range" if args.scaling == "weak"
                                  else f"a step = the whole stream, {B}-buffer batches") + " (inputs > L2 per step)",
                   "buffer_len": N, "buffers_per_step_per_gpu": B, "parallelism": f"buffer-sharded x{world}",
                   "stream_buffers": S, "pool": P,
                   "shards": [list(shard_range(S, world, r)) for r in range(world)],
                   "buffers_timed": tot["symbols"] // (N // 4)},
        "comm": comm_info(),
                   "l2": "inputs larger than L2: each step reads %d x %.0f MiB = %.0f MiB of int16 codes from "
                         "distinct device memory (the %d-buffer pool laid out cycled into a %d-buffer stream); "
                         "L2 is 126 MB" % (B, N * 2 / 2**20, B * N * 2 / 2**20, P, P + B),
        "gbaud_equiv": value / 4.0,
        "hbm_fraction": value * HBM_BYTES_PER_SA / hbm,
        "fp32_fraction_chain": value * FLOP_PER_SA_CHAIN / (FP32_PEAK_TFLOPS * 1e3),
        "roofline": {"bound": "alu", "kernel": "kk_chain_kernel<APPLY>", "achieved": achieved_tf,
                     "peak": FP32_PEAK_TFLOPS, "unit": "TFLOP/s", "frac": achieved_tf / FP32_PEAK_TFLOPS,
                     "traffic": (traffic["chain_dram_bytes_per_launch"] * (B * N) / traffic["chain_samples_per_launch"]
                                 if traffic else None),
                     "traffic_source": (traffic or {}).get("source"),
                     "flop_per_sa": FLOP_PER_SA_KERNEL, "samples_per_launch": B * N, "avg_launch_ms": ch_avg_ms,
                     "hbm_algorithmic_bytes_per_launch": HBM_BYTES_PER_SA * B * N,
                     "hbm_achieved_gbs": HBM_BYTES_PER_SA * B * N / (ch_avg_ms / 1e3) / 1e9,
                     "peak_basis": "148 SM x 128 FP32 lanes x 2 x 1.965 GHz (derived, DESIGN.md)",
                     "peak_measured_fp32": FP32_MEASURED_TFLOPS,
                     "peak_measured_basis": "FFMA throughput microbenchmark on this B200 (tools/microbench/f32x2_rate.cu: "
                                            "7.652 warp-FFMA/ns/SM x 32 lanes x 2 flop x 148 SMs)",
                     "frac_of_measured": achieved_tf / FP32_MEASURED_TFLOPS,
                     "issue_limit": issue_limit(traffic, B * N, ch_avg_ms)},
        "kernel_ms_per_step": {"chain": ch_avg_ms, "lms_overlapped": lms_avg},
        "pipeline": ("kk_rx_submit_batch per step + one kk_rx_sync: the LMS update pass of batch j (one SM, "
                     "lane-per-chain) overlaps the fused chain of batch j-1, whose launch also computes batch j's "
                     "update-pass x2 tails first"),
        "sync_value": samples_total / world / (sync_ms / 1e3) / 1e9 * world,
        "errors": {"bit_errors": tot["bit_errors"], "bits": tot["bits"], "ber": tot["bit_errors"] / max(tot["bits"], 1),
                   "reduced_over_ranks": "sharding.reduce_counts (all_reduce SUM over the process group)"},
        # context only (north star): the paper's receiver ran the chain in real time at 4 GSa/s
        # (1 GBaud, 4 sps, 12-bit 4 GS/s ADC) on one commercial GPU "with 5120 processing cores"
        # that it "almost fully utilizes"; another machine's number
        "paper_context": {"value": 4.0, "unit": UNIT, "gbaud": 1.0, "hardware": "commercial GPU, 5120 cores",
                          "cite": "PAPER.md l.25, l.47, l.68, l.167", "ratio": value / world / 4.0,
                          "note": "per-GPU value / the paper's real-time rate; context, not a baseline"},
        "gpu_launches": launches,
        "clocks": clk.summary(),
    }
    if e2e:
        line["e2e"] = e2e
    if cufft_cmp:
        line["cufft_comparison"] = cufft_cmp
    if world == 1 and not args.no_cpu_baseline:
        workers = args.ref_workers or (os.cpu_count() or 1)
        v, dt, s = oracle_rate(args.workload, P, workers, workers)
        line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": workers, "kind": "oracle", "cpu_model": cpu_model(),
                                "sample": f"{workers} whole 2^22-sample C5 buffers, one per process ({dt:.1f} s)"}
    print(json.dumps(line), flush=True)
    rx.close()
    if dist_on:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="kk", choices=["kk", "reference"])
    ap.add_argument("--workload", default="C5")
    ap.add_argument("--batch", type=int, default=128)
    ap.add_argument("--pool", type=int, default=64, help="distinct buffers of the cycled pool (C5: 64)")
    ap.add_argument("--stream", type=int, default=0, help="stream length in buffers (0 = the workload's: C5 4096)")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="weak: B buffers per GPU per step; strong: a step = the whole stream over all GPUs")
    ap.add_argument("--ref-workers", type=int, default=0, help="oracle processes (0 = all host cores)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-cufft", action="store_true", help="skip the cuFFT comparison leg")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3  # timing rule: W >= 3
    if args.impl == "reference":
        return run_reference(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
