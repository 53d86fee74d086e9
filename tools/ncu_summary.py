"""Summarise an ncu report: headline metrics, stall mix, top source lines.
usage: python tools/ncu_summary.py report.ncu-rep [n_lines]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
nl = int(sys.argv[2]) if len(sys.argv) > 2 else 30


def ncu(*args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


raw = list(csv.reader(io.StringIO(ncu("--page", "raw", "--csv"))))
h, v = raw[0], raw[2]
d = dict(zip(h, v))
keys = ["Kernel Name", "gpu__time_duration.sum", "smsp__inst_executed.sum", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "sm__cycles_elapsed.avg.per_second"]
for k in keys:
    print(f"{k:70s} {d.get(k)}")
st = {k: float(x) for k, x in d.items() if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued") and x}
tot = sum(st.values()) or 1
print("-- stall mix")
for k, x in sorted(st.items(), key=lambda t: -t[1])[:10]:
    print(f"  {x / tot * 100:5.1f}% {k.replace('smsp__pcsamp_warps_issue_stalled_', '')}")
rows = list(csv.reader(io.StringIO(ncu("--page", "source", "--csv", "--print-source", "cuda,sass"))))
cur, out, hdr = None, [], None
for r in rows:
    if r and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 9 or r[2] != "-":
        continue
    try:
        out.append((int(r[7]), int(r[6]), cur, r[0], r[1][:95]))
    except ValueError:
        pass
ti = sum(o[0] for o in out) or 1
ts = sum(o[1] for o in out) or 1
print(f"-- top source lines (instructions executed; stall samples), total inst {ti}")
for o in sorted(out, key=lambda t: -t[0])[:nl]:
    print(f"{o[0] / ti * 100:5.1f}% {o[1] / ts * 100:5.1f}%  {o[2]}:{o[3]}  {o[4]}")
