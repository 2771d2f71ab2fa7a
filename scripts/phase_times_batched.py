"""Per-CTA phase durations of the batched kernel (profiling build only)."""
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
                    "-fPIC", "-DDRS_PHASE_TIMING", *os.environ.get("DRS_PROF_FLAGS", "").split(), "-c",
                    str(csrc / f"{f}.cu"), "-o", o], check=True)
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
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
L = _lib.lib()
L.dr_debug_phase_times_batched.argtypes = [ctypes.c_void_p, ctypes.c_int]
for rep in range(4):
    flush.fill_(rep)
    drs.resample_batched(w, Nf, bs, return_uniforms=True, check=False, device=True)
    torch.cuda.synchronize()
nc = 2 * B
buf = np.zeros(nc * 16, dtype=np.uint64)
L.dr_debug_phase_times_batched(buf.ctypes.data, buf.size)
t = buf.reshape(nc, 16)[:, :6].astype(np.float64)
t0 = t[:, 0].min()
t = (t - t0) / 1e3
span = t[:, 5].max()
names = ["start", "(init)", "tile landed", "sweep+fold (+U copy issued)", "exchange (+U landed)", "s* + search + write"]
print(f"c4: {nc} CTAs, kernel span {span:.1f} us")
for k in range(1, 6):
    d = t[:, k] - t[:, k - 1]
    print(f"  {names[k]:18s} median {np.median(d):6.2f}  p90 {np.percentile(d, 90):6.2f}  max {d.max():6.2f} us")
life = t[:, 5] - t[:, 0]
print(f"  CTA lifetime      median {np.median(life):6.2f}  p90 {np.percentile(life, 90):6.2f}")
print(f"  mean concurrent CTAs = {life.sum() / span:.0f}")
