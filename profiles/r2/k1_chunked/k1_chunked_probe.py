"""Probe of the chunked single-kernel table build (dr_build_table_chunked,
prototype): S and T bit-exact against the oracle's device association, and
its time against the two-pass build at c3 for several chunk sizes."""
import ctypes
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
from oracle import oracle as orc  # noqa: E402
from paper_2604_01356_b200 import _lib  # noqa: E402
import paper_2604_01356_b200 as drs  # noqa: E402

L = _lib.lib()
V = ctypes.c_void_p
L.dr_build_table_chunked.argtypes = [V, ctypes.c_int64, V, V, V, V, ctypes.c_int64, V, ctypes.c_size_t, V]
L.dr_build_table_chunked.restype = ctypes.c_int


def build(w, ct):
    m = w.numel()
    S = torch.empty(m, dtype=torch.float64, device="cuda")
    n = int(L.dr_index_entries(m))
    idx = torch.empty(max(n, 1), dtype=torch.float64, device="cuda")
    OT = torch.empty(2, dtype=torch.float64, device="cuda")
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    ws, wsb = _lib.workspace(L.dr_workspace_bytes(_lib.OP_TABLE, m, 0, 0))
    rc = L.dr_build_table_chunked(w.data_ptr(), m, S.data_ptr(), idx.data_ptr() if n else 0, OT.data_ptr(),
                                  st.data_ptr(), ct, ws, wsb, _lib.stream_handle())
    assert rc == 0, rc
    return S, OT, st


for M in (1, 33, 8449, 32 * 8448 + 5, 1 << 20, (1 << 22) + 3):
    w = np.random.default_rng(M).random(M) + 0.01
    for ct in (32, 64, 0):
        S, OT, st = build(torch.from_numpy(w).cuda(), ct)
        So, To = orc.chain_scan(w, 33)
        ok = np.array_equal(S.cpu().numpy(), So) and OT.cpu().tolist() == [0.0, To] and int(st.item()) == 0
        print(f"M={M} ct={ct} exact={ok}")
        assert ok
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
w = torch.from_numpy(bench.make_weights("c3")).cuda()


def timed(fn, k=15):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(k):
        flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return float(np.median(ts))


print(f"c3 two-pass: {timed(lambda: drs.build_weight_table(w, check=False)):.1f} us")
for ct in (444, 888, 1332, 1776, 2664):
    print(f"c3 chunked ct={ct} ({ct * 8448 * 8 / 2**20:.0f} MB of w): {timed(lambda: build(w, ct)):.1f} us")
S, OT, st = build(w, 888)
So, To = orc.chain_scan(w.cpu().numpy(), 33)
print("c3 exact:", np.array_equal(S.cpu().numpy(), So), OT.cpu().tolist()[1] == To)
