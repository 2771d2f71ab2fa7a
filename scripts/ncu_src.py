"""Per-source-line instructions and stall reasons of one kernel in an ncu report.

  python scripts/ncu_src.py REPORT.ncu-rep [kernel-regex] [top]
"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
kre = sys.argv[2] if len(sys.argv) > 2 else None
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"]
if kre:
    cmd[3:3] = ["--kernel-name", f"regex:{kre}"]
rows = list(csv.reader(io.StringIO(subprocess.run(cmd, capture_output=True, text=True).stdout)))
hdr, per, tot = None, [], collections.Counter()
for r in rows:
    if len(r) > 4 and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr) or not r[0]:
        continue
    d = dict(zip(hdr, r))
    try:
        s, ins = int(d["Warp Stall Sampling (All Samples)"]), int(d["Instructions Executed"])
    except ValueError:
        continue
    st = {k[6:]: int(v) for k, v in d.items() if k.startswith("stall_") and "Not Issued" not in k and v.isdigit()}
    tot.update(st)
    per.append((s, ins, r[0], r[1].strip()[:64], st))
T = sum(tot.values()) or 1
TI = sum(p[1] for p in per) or 1
print(f"warp instructions {TI}, stall samples {T}")
print("stalls:", {k: round(100 * v / T, 1) for k, v in tot.most_common(10)})
for s, ins, ln, src, st in sorted(per, key=lambda p: (p[0], p[1]), reverse=True)[:top]:
    t3 = sorted(st.items(), key=lambda x: -x[1])[:3]
    print(f"{100*s/T:5.1f}%s {100*ins/TI:5.1f}%i L{ln:>4} {src:64s} {t3}")
