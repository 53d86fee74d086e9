"""Per-source-line instructions and stall breakdown of an ncu report (source page).
usage: python tools/ncu_lines.py report.ncu-rep [n_lines] [--regions]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
nl = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
cur, hdr, recs = None, None, []
for r in rows:
    if not r:
        continue
    if r[0] == "File Path" or r[0] == "File Name":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr) or r[2] != "-":
        continue
    d = dict(zip(hdr[2:], r[2:]))
    d["Line No"], d["Source"] = r[0], r[1]
    try:
        inst = int(d["Instructions Executed"] or 0)
        samp = int(d["Warp Stall Sampling (All Samples)"] or 0)
    except ValueError:
        continue
    st = {k[6:]: int(v or 0) for k, v in d.items() if k.startswith("stall_") and "Not Issued" not in k and v not in ("", "0")}
    recs.append((cur, int(d["Line No"]), d["Source"].strip()[:80], inst, samp, st))
ti = sum(r[3] for r in recs) or 1
ts = sum(r[4] for r in recs) or 1
tot = {}
for r in recs:
    for k, v in r[5].items():
        tot[k] = tot.get(k, 0) + v
print("total inst", ti, "samples", ts, " ".join(f"{k}={v/ts*100:.1f}%" for k, v in sorted(tot.items(), key=lambda t: -t[1])[:10]))
for r in sorted(recs, key=lambda t: -t[4])[:nl]:
    top = sorted(r[5].items(), key=lambda t: -t[1])[:4]
    print(f"{r[0]}:{r[1]:<4d} inst {r[3]/ti*100:5.1f}% samp {r[4]/ts*100:5.1f}%  " +
          " ".join(f"{k}:{v/max(r[4],1)*100:.0f}" for k, v in top) + f"   | {r[2]}")
