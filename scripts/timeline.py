"""Kernel timeline of one sampler step (profiling build only).

Builds libdrs with -DDRS_PHASE_TIMING into /tmp, runs one public sampler
call of a bench config after an L2 flush, and prints, for every kernel that
stamped (STAMPK), its CTA count and, relative to the first CTA entry of the
step (us): first entry, median/max "dependency satisfied", median/max exit,
plus the events around the call.

    python scripts/timeline.py c2 dac auto
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
so = Path("/tmp/libdrs_tl.so")
objs = []
for f in sorted(x.stem for x in csrc.glob("*.cu")):
    o = f"/tmp/{f}_tl.o"
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-Xcompiler",
                    "-fPIC", "-DDRS_PHASE_TIMING", "-c", str(csrc / f"{f}.cu"), "-o", o], check=True)
    objs.append(o)
subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-cudart", "static", "-o",
                str(so)] + objs, check=True)

from paper_2604_01356_b200 import _lib  # noqa: E402

_lib.LIB_PATH = so
import bench  # noqa: E402
import paper_2604_01356_b200 as drs  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
sampler = sys.argv[2] if len(sys.argv) > 2 else "dac"
mode = sys.argv[3] if len(sys.argv) > 3 else "auto"
c = bench.CONFIGS[cfg]
L = _lib.lib()
TUS = {"scan": ["pass1", "chain", "pass2", "finalize", "table_local", "table_levels", "k6", "tail_phases"],
       "match": ["k0", "k1", "k2", "k3", "merge_tiles", "merge_heavy", "top_guide", "k7"],
       "": ["k0", "k1", "k2", "k3", "k4", "k5", "finish", "k7"]}
for tu in TUS:
    sfx = f"_{tu}" if tu else ""
    getattr(L, f"dr_debug_phase_times{sfx}").argtypes = [ctypes.c_void_p, ctypes.c_int]
table = drs.build_weight_table(bench.make_weights(cfg))
N = c["N"]
if sampler == "table":  # K1 (build_weight_table, single pass) from device weights
    w_dev = torch.from_numpy(bench.make_weights(cfg)).cuda()
    fn = lambda table, N, st, device, out, **kw: drs.build_weight_table(w_dev, check=False)  # noqa: E731
else:
    fn = {"dac": drs.dac_sampler, "ccf": drs.ccf_sampler, "binary": drs.binary_sampler}[sampler]
kw = {"mode": mode} if sampler == "dac" else {}
out = torch.empty(N, dtype=torch.int64, device="cuda")
if sampler not in ("binary", "table"):
    kw["uniforms_out"] = torch.empty(N, dtype=torch.float64, device="cuda")
st = drs.RngStream(c["useed"])
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for rep in range(4):
    fn(table, N, st, device=True, out=out, **kw)
torch.cuda.synchronize()
for tu in TUS:
    getattr(L, f"dr_debug_phase_clear{'_' + tu if tu else ''}")()
flush.fill_(3)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
fn(table, N, st, device=True, out=out, **kw)
e1.record()
torch.cuda.synchronize()
rows = []
for tu, names in TUS.items():
    buf = np.zeros(8 * 65536 * 4, dtype=np.uint64)
    getattr(L, f"dr_debug_phase_times{'_' + tu if tu else ''}")(buf.ctypes.data, buf.size)
    t = buf.reshape(8, 65536, 4).astype(np.float64)
    for k in range(8):
        if tu == "" and k != 6:
            continue  # k_dac_fused stamps with the older per-phase layout (scripts/phase_times.py); k_finish_search is k = 6
        ent = t[k, :, 0]
        live = ent > 0
        if live.any():
            rows.append((names[k], t[k][live]))
t0 = min(r[1][:, 0].min() for r in rows)
print(f"{cfg} {sampler} {mode}: events around the call {e0.elapsed_time(e1) * 1e3:.2f} us; times since the first CTA entry (us)")
print(f"  {'kernel':14s} {'CTAs':>6s} {'entry0':>8s} {'entry_med':>9s} {'dep_med':>8s} {'dep_max':>8s} {'work_med':>8s} {'work_max':>8s} {'exit_med':>8s} {'exit_max':>8s}")
for name, v in sorted(rows, key=lambda r: r[1][:, 0].min()):
    rel = np.where(v > 0, (v - t0) / 1e3, np.nan)
    w = rel[:, 2] if np.isfinite(rel[:, 2]).any() else np.full(rel.shape[0], np.nan)
    print(f"  {name:14s} {v.shape[0]:6d} {np.nanmin(rel[:, 0]):8.2f} {np.nanmedian(rel[:, 0]):9.2f} {np.nanmedian(rel[:, 1]):8.2f} "
          f"{np.nanmax(rel[:, 1]):8.2f} {np.nanmedian(w):8.2f} {np.nanmax(w):8.2f} {np.nanmedian(rel[:, 3]):8.2f} {np.nanmax(rel[:, 3]):8.2f}")
