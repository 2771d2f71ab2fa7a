"""Phase stamps of the one-CTA tile chain k_chain_groups for the c3 table (profiling build)."""
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

w = torch.from_numpy(bench.make_weights("c3")).cuda()
L = _lib.lib()
L.dr_debug_phase_times_scan.argtypes = [ctypes.c_void_p, ctypes.c_int]
for rep in range(3):
    drs.build_weight_table(w)
    torch.cuda.synchronize()
buf = np.zeros(16, dtype=np.uint64)
L.dr_debug_phase_times_scan(buf.ctypes.data, buf.size)
t = (buf[:6].astype(np.float64) - float(buf[0])) / 1e3
names = ["entry", "staged", "group folds", "incl written", "C fold", "grp written"]
for k in range(1, 6):
    print(f"  {names[k]:14s} +{t[k] - t[k - 1]:6.2f} us  (at {t[k]:6.2f})")
