"""Per-source-line stall samples and executed instructions from an ncu report.

  python scripts/ncu_lines.py REPORT.ncu-rep [top]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = None
lines = []
for r in rows:
    if len(r) > 4 and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr) or not r[0]:
        continue
    d = dict(zip(hdr, r))
    try:
        samp = int(d["Warp Stall Sampling (All Samples)"])
        inst = int(d["Instructions Executed"])
    except ValueError:
        continue
    lines.append((samp, inst, r[0], r[1].strip()[:90]))
tot_s = sum(x[0] for x in lines) or 1
tot_i = sum(x[1] for x in lines) or 1
print(f"total samples {tot_s}, warp instructions {tot_i}")
for s, i, ln, src in sorted(lines, reverse=True)[:top]:
    print(f"{100*s/tot_s:5.1f}% samp {100*i/tot_i:5.1f}% inst  L{ln:>4} {src}")
