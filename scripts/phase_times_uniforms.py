"""Per-warp phase times of the batched uniforms kernel (profiling build; config c4).

One warp per filter: start, keys loaded, Philox words, logs, row folds, U
stored.  Prints the medians of each phase and the spread of warp start times.
"""
import ctypes
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
                    "-fPIC", "-DDRS_PHASE_TIMING", "-c", str(csrc / f"{f}.cu"), "-o", o], check=True)
    objs.append(o)
subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-cudart", "static", "-o",
                str(so)] + objs, check=True)
from paper_2604_01356_b200 import _lib  # noqa: E402

_lib.LIB_PATH = so
import paper_2604_01356_b200 as drs  # noqa: E402
import bench  # noqa: E402

c = bench.CONFIGS["c4"]
w = torch.from_numpy(bench.make_weights("c4")).cuda()
B, Nf = w.shape[0], c["Nf"]
bs = drs.BatchedStreams([drs.RngStream(c["useed"], (b,)) for b in range(B)])
L = _lib.lib()
L.dr_debug_phase_times_batched.argtypes = [ctypes.c_void_p, ctypes.c_int]
for rep in range(3):
    torch.cuda.synchronize()
    torch.cuda._sleep(2_000_000)  # an idle-ish GPU before the measured call (a spinning single-thread kernel)
    drs.resample_batched(w, Nf, bs, return_uniforms=True, check=False, device=True)
    torch.cuda.synchronize()
buf = np.zeros(150000 + B * 8, dtype=np.uint64)  # the uniforms' stamps start at 150000 (after the cluster kernel's)
L.dr_debug_phase_times_batched(buf.ctypes.data, buf.size)
t = buf[150000:].reshape(B, 8)[:, :6].astype(np.float64)
t0 = t[:, 0].min()
t = (t - t0) / 1e3
names = ["start", "keys", "philox", "logs", "row folds", "U stored"]
print(f"uniforms: {B} warps, span {t[:, 5].max():.1f} us; warp start: median {np.median(t[:, 0]):.2f} p90 "
      f"{np.percentile(t[:, 0], 90):.2f} max {t[:, 0].max():.2f} us")
for k in range(1, 6):
    d = t[:, k] - t[:, k - 1]
    print(f"  {names[k]:10s} median {np.median(d):6.2f}  p90 {np.percentile(d, 90):6.2f}  max {d.max():6.2f} us")
life = t[:, 5] - t[:, 0]
print(f"  warp lifetime median {np.median(life):.2f} us")
ev = np.concatenate([np.stack([t[:, 0], np.ones(B)], 1), np.stack([t[:, 5], -np.ones(B)], 1)])
ev = ev[np.argsort(ev[:, 0], kind="stable")]
conc = np.cumsum(ev[:, 1])
print(f"  max concurrent warps {conc.max():.0f}; warps started in the first 2 us: {(t[:, 0] < 2).sum()}")
order = np.argsort(t[:, 0])
print("  start times by launch index (warp 0, 512, 1024, ... 3584):",
      " ".join(f"{t[i, 0]:.1f}" for i in range(0, B, 512)))
