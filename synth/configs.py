"""Named workloads (BASELINE.json configs C1-C5) and small
test-size variants.  Seeds: seed_pat = 1, seed_noise = 1000 + config number.

C1  MP 4-QAM, CSPR 12 dB (PAPER l.77 inset), noiseless, 1 buffer
C2  MP 16-QAM, CSPR 14 dB, one-sided AWGN at OSNR 20 dB, 16 buffers
C3  8-QAM / GS-8 (OSNR 8-14, CSPR 6-12) and 32-QAM (OSNR 18-24, CSPR 10-16),
    two-sided noise, 4x4 grid x 4 buffers = 64 buffers per format
C4  MP 64-QAM, CSPR 16 dB, two-sided at OSNR 28.2 dB, 256 buffers
C5  GS-128, CSPR 16 dB, two-sided at OSNR 35 dB, 64-buffer pool cycled to a
    4096-buffer stream (the throughput workload)
"""
from __future__ import annotations

from dataclasses import dataclass, replace

from .generate import LinkConfig

N_FULL = 1 << 22
N_SMALL = 1 << 16


@dataclass(frozen=True)
class Workload:
    name: str
    link: LinkConfig
    n_buffers: int
    n_pool: int


def _c3_cells():
    out = []
    for fmt in ("QAM8", "GS8"):
        for osnr in (8.0, 10.0, 12.0, 14.0):
            for cspr in (6.0, 8.0, 10.0, 12.0):
                out.append((fmt, cspr, osnr))
    for osnr in (18.0, 20.0, 22.0, 24.0):
        for cspr in (10.0, 12.0, 14.0, 16.0):
            out.append(("QAM32", cspr, osnr))
    return out


def workloads(buffer_len=N_FULL):
    sfx = "" if buffer_len == N_FULL else "_n%d" % (buffer_len.bit_length() - 1)
    w = {}
    w["C1" + sfx] = Workload("C1" + sfx, LinkConfig("QAM4", 12.0, None, "one_sided", buffer_len, seed_noise=1001), 1, 1)
    w["C2" + sfx] = Workload("C2" + sfx, LinkConfig("QAM16", 14.0, 20.0, "one_sided", buffer_len, seed_noise=1002), 16, 16)
    for fmt, cspr, osnr in _c3_cells():
        nm = "C3_%s_c%g_o%g%s" % (fmt, cspr, osnr, sfx)
        w[nm] = Workload(nm, LinkConfig(fmt, cspr, osnr, "two_sided", buffer_len, seed_noise=1003), 4, 4)
    w["C4" + sfx] = Workload("C4" + sfx, LinkConfig("QAM64", 16.0, 28.2, "two_sided", buffer_len, seed_noise=1004), 256, 256)
    w["C5" + sfx] = Workload("C5" + sfx, LinkConfig("GS128", 16.0, 35.0, "two_sided", buffer_len, seed_noise=1005), 4096, 64)
    return w


ALL = {}
ALL.update(workloads(N_FULL))
ALL.update(workloads(N_SMALL))


def get(name: str) -> Workload:
    return ALL[name]


def with_buffers(wl: Workload, n_buffers: int, n_pool: int | None = None) -> Workload:
    return replace(wl, n_buffers=n_buffers, n_pool=n_pool if n_pool is not None else min(wl.n_pool, n_buffers))
