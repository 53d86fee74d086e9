"""Summarise an `ncu --set full` report of the chain kernel for profiles/ and (optionally)
refresh profiles/traffic.json, which bench.py reads for roofline.traffic / issue_limit.

    python tools/ncu_summary.py REPORT.ncu-rep OUT.txt [--traffic profiles/traffic.json --samples S --cmd "..."]

--samples: ADC samples the captured launch processed (buffers x 2^22; required with --traffic).
"""
import csv
import io
import json
import subprocess
import sys

rep, out = sys.argv[1], sys.argv[2]
traffic = sys.argv[sys.argv.index("--traffic") + 1] if "--traffic" in sys.argv else None
cmd = sys.argv[sys.argv.index("--cmd") + 1] if "--cmd" in sys.argv else "?"
samples = int(sys.argv[sys.argv.index("--samples") + 1]) if "--samples" in sys.argv else None
if traffic and not samples:
    sys.exit("--traffic needs --samples (samples processed by the captured launch)")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
d = dict(zip(hdr, vals))
u = dict(zip(hdr, units))
keys = ["Kernel Name", "gpu__time_duration.sum", "smsp__inst_executed.sum", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "sm__cycles_elapsed.avg.per_second"]
lines = [f"{k:<70s} {d.get(k, '?')} {u.get(k, '')}".rstrip() for k in keys]
stall = {k: float(d[k]) for k in hdr if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")
         and d.get(k, "") not in ("", "n/a")}
tot = sum(stall.values()) or 1.0
lines.append("-- stall mix (pc sampling)")
for k, v in sorted(stall.items(), key=lambda t: -t[1])[:10]:
    lines.append(f"  {v / tot * 100:5.1f}% {k.replace('smsp__pcsamp_warps_issue_stalled_', '')}")
src = subprocess.run([sys.executable, __file__.replace("ncu_summary.py", "ncu_lines.py"), rep, "25"],
                     capture_output=True, text=True).stdout
lines.append("-- top source lines (tools/ncu_lines.py: instructions executed %, stall samples %)")
lines += src.rstrip().split("\n")
open(out, "w").write("\n".join(lines) + "\n")
print("\n".join(lines[:20]))


def mb(k):
    v = float(d[k].replace(",", ""))
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u[k], 1)


if traffic:
    t = json.load(open(traffic))
    rd, wr = mb("dram__bytes_read.sum"), mb("dram__bytes_write.sum")
    t["chain_dram_bytes_per_launch"] = int(rd + wr)
    t["chain_samples_per_launch"] = samples
    t["chain_algorithmic_bytes_per_launch"] = int(2.25 * samples)
    t["chain_warp_inst_per_launch"] = int(float(d["smsp__inst_executed.sum"]))
    t["source"] = (f"ncu --set full of the timed combined kk_chain_kernel launch of `{cmd}`: dram__bytes_read.sum "
                   f"{rd / 1e6:.6f} MB + dram__bytes_write.sum {wr / 1e6:.6f} MB; {out}")
    t["inst_source"] = f"smsp__inst_executed.sum of the same capture ({out})"
    json.dump(t, open(traffic, "w"), indent=2)
    print("traffic.json updated:", t["chain_dram_bytes_per_launch"], t["chain_warp_inst_per_launch"])
