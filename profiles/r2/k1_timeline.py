"""Phase timeline of the single-pass table scan at c3 (profiling build)."""
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

L = _lib.lib()
V = ctypes.c_void_p
L.dr_build_table_s.argtypes = [V, ctypes.c_int64, V, V, V, V, V, ctypes.c_size_t, V]
L.dr_debug_phase_times_scan.argtypes = [V, ctypes.c_int]
w = torch.from_numpy(bench.make_weights(sys.argv[1] if len(sys.argv) > 1 else "c3")).cuda()
m = w.numel()
S = torch.empty(m, dtype=torch.float64, device="cuda")
n = int(L.dr_index_entries(m))
idx = torch.empty(max(n, 1), dtype=torch.float64, device="cuda")
OT = torch.empty(2, dtype=torch.float64, device="cuda")
st = torch.zeros(1, dtype=torch.int32, device="cuda")
ws, wsb = _lib.workspace(L.dr_workspace_bytes(_lib.OP_TABLE, m, 0, 0))
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for rep in range(4):
    flush.fill_(rep)
    L.dr_debug_phase_clear_scan()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    L.dr_build_table_s(w.data_ptr(), m, S.data_ptr(), idx.data_ptr(), OT.data_ptr(), st.data_ptr(), ws, wsb,
                       _lib.stream_handle())
    e1.record()
    torch.cuda.synchronize()
buf = np.zeros(8 * 65536 * 4, dtype=np.uint64)
L.dr_debug_phase_times_scan(buf.ctypes.data, buf.size)
t = buf.reshape(8, 65536, 4).astype(np.float64)
nt = (m + 8447) // 8448
k6 = t[6, :nt]
ex = t[7, :nt, 3]
t0 = k6[:, 0].min()
rel = (k6 - t0) / 1e3
rex = (ex - t0) / 1e3
print(f"events {e0.elapsed_time(e1) * 1e3:.1f} us; {nt} CTAs (blockIdx order); us since first entry")
names = ["entry", "id+gen", "A published", "C known"]
for k in range(4):
    print(f"  {names[k]:12s} min {rel[:, k].min():7.2f} med {np.median(rel[:, k]):7.2f} max {rel[:, k].max():7.2f}")
print(f"  {'exit':12s} min {rex.min():7.2f} med {np.median(rex):7.2f} max {rex.max():7.2f}")
life = rex - rel[:, 0]
print("  CTA lifetime   med %.2f p90 %.2f max %.2f" % (np.median(life), np.percentile(life, 90), life.max()))
for nm, a, b in (("id wait", 0, 1), ("load+reduce", 1, 2), ("lookback", 2, 3)):
    dd = rel[:, b] - rel[:, a]
    print(f"  {nm:12s} med {np.median(dd):6.2f} p90 {np.percentile(dd, 90):6.2f} max {dd.max():6.2f}")
dd = rex - rel[:, 3]
print(f"  {'S+store':12s} med {np.median(dd):6.2f} p90 {np.percentile(dd, 90):6.2f} max {dd.max():6.2f}")

k5 = t[5, :nt]
dd = (k5[:, 0] - k6[:, 2]) / 1e3
print(f"  D wait       med {np.median(dd):6.2f} p90 {np.percentile(dd, 90):6.2f} max {dd.max():6.2f}")
ok = k5[:, 1] > 0
dd = (k5[ok, 1] - k5[ok, 0]) / 1e3
print(f"  C base scan  med {np.median(dd):6.2f} p90 {np.percentile(dd, 90):6.2f} max {dd.max():6.2f}")
dd = (k6[ok, 3] - k5[ok, 1]) / 1e3
print(f"  E fold       med {np.median(dd):6.2f} p90 {np.percentile(dd, 90):6.2f} max {dd.max():6.2f}")
dist = t[4, :nt, 0][ok]
print(f"  g - b        med {np.median(dist):6.1f} p90 {np.percentile(dist, 90):6.1f} max {dist.max():6.1f}")
# which tile id did each CTA get?  (ids come from the counter; blockIdx order roughly equals id order)
