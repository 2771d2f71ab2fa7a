"""Summarise ncu captures into small JSON files for profiles/.

  python scripts/ncu_summary.py OUT.json REPORT.ncu-rep [REPORT2.ncu-rep ...]
  python scripts/ncu_summary.py --launches OUT.json LAUNCHES.csv

For a --set full report: per kernel launch, duration, DRAM bytes, achieved
DRAM GB/s, SM/memory throughput, occupancy and launch geometry.
For a launch list (--metrics gpu__time_duration.sum): every launch in order
plus per-kernel totals and shares.
"""

from __future__ import annotations

import csv
import io
import json
import subprocess
import sys
from collections import OrderedDict

KEYS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_bytes.sum",
    "launch__grid_size",
    "launch__block_size",
    "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum",
]

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "us": 1e-6, "ms": 1e-3, "ns": 1e-9, "s": 1,
         "msecond": 1e-3, "usecond": 1e-6, "nsecond": 1e-9}


def _num(v, unit):
    try:
        x = float(v.replace(",", ""))
    except ValueError:
        return v
    return x * SCALE.get(unit, 1)


def full(report):
    raw = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        e = OrderedDict(kernel=d.get("Kernel Name", ""))
        for k in KEYS:
            if k in hdr:
                e[k] = _num(d[k], units[hdr.index(k)])
        t = e.get("gpu__time_duration.sum")
        if isinstance(t, float) and t > 0:
            rd = e.get("dram__bytes_read.sum", 0) or 0
            wr = e.get("dram__bytes_write.sum", 0) or 0
            e["dram_bytes"] = rd + wr
            e["dram_GBps"] = (rd + wr) / t / 1e9
            e["duration_us"] = t * 1e6
        out.append(e)
    return out


def launches(path):
    text = open(path).read()
    start = text.find('"ID"')
    rows = list(csv.reader(io.StringIO(text[start:])))
    hdr = rows[0]
    seq, tot = [], OrderedDict()
    for r in rows[1:]:
        if len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        ns = _num(d["Metric Value"], d.get("Metric Unit", "ns")) * (1 if d.get("Metric Unit") in SCALE else 1e-9)
        name = d["Kernel Name"]
        seq.append({"kernel": name, "us": ns * 1e6})
        t = tot.setdefault(name, {"launches": 0, "us": 0.0})
        t["launches"] += 1
        t["us"] += ns * 1e6
    all_us = sum(v["us"] for v in tot.values())
    for v in tot.values():
        v["share"] = v["us"] / all_us if all_us else 0.0
    return {"launches": seq, "per_kernel": tot}


def main():
    a = sys.argv[1:]
    if a and a[0] == "--launches":
        json.dump(launches(a[2]), open(a[1], "w"), indent=1)
        return
    res = {}
    for rep in a[1:]:
        res[rep.split("/")[-1]] = full(rep)
    json.dump(res, open(a[0], "w"), indent=1)


if __name__ == "__main__":
    main()
