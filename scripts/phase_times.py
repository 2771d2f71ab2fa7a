"""Phase breakdown of the fused dac_sampler kernel (profiling build only).

Builds libdrs with -DDRS_PHASE_TIMING into /tmp, runs dac_sampler on the c3
workload (L2 flushed before the measured call) and prints, per phase, the
median and max over CTAs of the time since the earliest CTA start (us).
"""
import ctypes
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
csrc = ROOT / "paper_2604_01356_b200" / "csrc"
so = Path("/tmp/libdrs_prof.so")
objs = []
for f in sorted(x.stem for x in csrc.glob("*.cu")):
    o = f"/tmp/{f}_prof.o"
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-Xcompiler",
                    "-fPIC", "-DDRS_PHASE_TIMING", *os.environ.get("DRS_PROF_FLAGS", "").split(), "-c", str(csrc / f"{f}.cu"), "-o", o], check=True)
    objs.append(o)
subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-cudart", "static", "-o",
                str(so)] + objs, check=True)

from paper_2604_01356_b200 import _lib  # noqa: E402

_lib.LIB_PATH = so
import paper_2604_01356_b200 as drs  # noqa: E402
import bench  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
c = bench.CONFIGS[cfg]
table = drs.build_weight_table(bench.make_weights(cfg), deferred=os.environ.get("DRS_TABLE", "deferred") == "deferred")
N = c["N"]
st = drs.RngStream(c["useed"])
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
L = _lib.lib()
L.dr_debug_phase_times.argtypes = [ctypes.c_void_p, ctypes.c_int]
names = ["start", "draws+log", "tile fold", "grid barrier", "chain fold", "U", "index staged", "search", "written"]
rows = []
for rep in range(6):
    if not os.environ.get("NOFLUSH"):
        flush.fill_(rep)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if os.environ.get("SMEM_PRIME"):
        drs.binary_sampler(table, 1, drs.RngStream(1), device=True)  # a big-smem kernel before the timed call
    e0.record()
    out = drs.dac_sampler(table, N, st, device=True)
    e1.record()
    torch.cuda.synchronize()
    ev_us = e0.elapsed_time(e1) * 1e3
    nt = (N + 1 + 511) // 512
    buf = np.zeros(nt * 16, dtype=np.uint64)
    L.dr_debug_phase_times(buf.ctypes.data, buf.size)
    t = buf.reshape(nt, 16)[:, :16].astype(np.float64)
    base = t[:, 10].min() if t[:, 10].min() > 0 else t[:, 0].min()
    rows.append(np.where(t > 0, t - base, 0.0))
t = rows[-1]
print(f"{cfg}: {t.shape[0]} CTAs; times since the first CTA entered (us): median / max over CTAs; events around the call {ev_us:.2f} us")
for k, nm in enumerate(names):
    print(f"  {k} {nm:14s} {np.median(t[:, k]) / 1e3:8.2f} {t[:, k].max() / 1e3:8.2f}")
for k, nm in [(10, "entry"), (9, "all arrived"), (13, "C fold"), (11, "lvl3 (smem)"), (12, "lvl2 (L2)"), (14, "lvl1")]:
    if t[:, k].max() > 0:
        print(f"  {k} {nm:14s} {np.median(t[:, k]) / 1e3:8.2f} {t[:, k].max() / 1e3:8.2f}")
