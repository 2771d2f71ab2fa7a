"""A/B of dr_build_table_deferred's tail: k_table_tail (chain + levels in one
launch) against k_chain_groups + k_table_levels (DRS_NO_TABLE_TAIL=1): the
table bytes must be identical; K1 timed by events with L2 flushed."""
import os
import statistics
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
import paper_2604_01356_b200 as drs  # noqa: E402


def build(w, tail):
    if tail:
        os.environ.pop("DRS_NO_TABLE_TAIL", None)
    else:
        os.environ["DRS_NO_TABLE_TAIL"] = "1"
    return drs.build_weight_table(w, check=True, deferred=True)


def arrays(t):
    out = []
    for name in ("_W", "_idx", "values", "index"):
        a = getattr(t, name, None)
        if isinstance(a, torch.Tensor):
            out.append(a.clone())
    return out


rng = np.random.default_rng(7)
ok = True
for M in (262145, 300000, (1 << 20) + 3, (1 << 22) + 5, 8448 * 4097, 1 << 26, 16384 * 8448, 16384 * 8448 + 1):
    w = torch.from_numpy(np.exp(2 * rng.standard_normal(M))).cuda()
    if M % 3 == 0:
        w[: M // 5] = 0.0
    a = build(w, True)
    b = build(w, False)
    ta, tb = arrays(a), arrays(b)
    assert len(ta) >= 2, [n for n in dir(a) if not n.startswith("__")]
    same = all(torch.equal(x.view(torch.int64), y.view(torch.int64)) for x, y in zip(ta, tb))
    print(f"M={M}: {len(ta)} arrays, identical={same}", flush=True)
    ok &= same
    del w, a, b, ta, tb
    torch.cuda.empty_cache()

w = torch.from_numpy(bench.make_weights("c3")).cuda()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for tail in (True, False, True, False):
    ms = []
    for r in range(25):
        flush.fill_(r)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        if tail:
            os.environ.pop("DRS_NO_TABLE_TAIL", None)
        else:
            os.environ["DRS_NO_TABLE_TAIL"] = "1"
        t = drs.build_weight_table(w, check=False, deferred=True)
        b.record()
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    print(f"c3 K1 tail={tail}: median {1e3 * statistics.median(ms[5:]):.1f} us, min {1e3 * min(ms[5:]):.1f} us", flush=True)
print("AB", "OK" if ok else "MISMATCH")
