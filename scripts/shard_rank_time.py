"""Per-rank device time of the W-sharded sampler (config 5), measured on ONE GPU.

For G in {1, 2, 4, 8} the G shards of the M = 2^30 table are built on this
GPU; then, for every rank g, its sampling kernels are timed by CUDA events
(L2 flushed): tile totals of its 1/G of the spacing tiles, the local chain +
regeneration of its own tiles (dr_shard_unif_local) and the match against its
shard.  The all-gather of the tile totals (2 * ceil(nt/G) doubles per rank)
is NOT included -- no NCCL here -- and no kernel waits on another rank: this
is the work split, not a multi-GPU measurement.  Also per rank: the shard's
table build (scan + finalize; the all-gather of the 24-byte totals excluded),
single-pass (deferred) and the two-pass legacy path (dr_shard_scan + dr_shard_finalize).
Prints one JSON line.
"""
import json
import statistics
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
import paper_2604_01356_b200 as drs  # noqa: E402
from paper_2604_01356_b200 import _lib as dlib  # noqa: E402
from paper_2604_01356_b200.sharded import DeviceShardOps, ShardedWeightTable, slice_capacity  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c5"
c = bench.CONFIGS[cfg]
M, N = c["M"], c["N"]
w = torch.from_numpy(bench.make_weights(cfg)).cuda()
import os  # noqa: E402

ops = DeviceShardOps(deferred=os.environ.get("DRS_SHARD_TABLE", "deferred") == "deferred")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
k0, k1 = drs.RngStream(c["useed"]).key


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    ts = []
    for r in range(reps):
        flush.fill_(r)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


res = {"config": cfg, "M": M, "N": N, "shards": "deferred" if ops.deferred else "two-pass",
       "note": __doc__.split("\n\n")[1].replace("\n", " ")}
ts = ops.tile_size()
nt = (N + 1 + ts - 1) // ts
for G in (1, 2, 4, 8):
    parts = [w[M * g // G: M * (g + 1) // G] for g in range(G)]
    scans = [ops.shard_scan(p) for p in parts]
    totals = torch.cat([s[1] for s in scans])
    tabs = []
    for g in range(G):
        W, idx = ops.finalize(scans[g][0], totals, G, g)
        tabs.append(ShardedWeightTable(W=W, index=idx, totals=totals, sizes=[p.numel() for p in parts], rank=g,
                                       world=G, totals_host=totals.cpu().tolist()))
    del scans
    bounds = [nt * h // G for h in range(G + 1)]
    shares = [ops.unif_tile_totals((k0, k1), 0, N, bounds[h], bounds[h + 1]) for h in range(G)]
    agg_all = torch.cat([a for a, _ in shares])
    zmin_all = torch.cat([z for _, z in shares])
    Lb = dlib.lib()

    def legacy_build(p, g):  # dr_shard_scan (two passes, raw S) + dr_shard_finalize (read/write + index pass)
        m = p.numel()
        S = torch.empty(m, dtype=torch.float64, device="cuda")
        Tg = torch.zeros(1, dtype=torch.float64, device="cuda")
        st = torch.zeros(1, dtype=torch.int32, device="cuda")
        idx = torch.empty(int(Lb.dr_index_entries(m)), dtype=torch.float64, device="cuda")
        ws, wsb = dlib.workspace(Lb.dr_workspace_bytes(dlib.OP_TABLE, m, 0, 0))
        dlib.check(Lb.dr_shard_scan(p.data_ptr(), m, S.data_ptr(), Tg.data_ptr(), st.data_ptr(), ws, wsb,
                                        dlib.stream_handle()), "dr_shard_scan")
        dlib.check(Lb.dr_shard_finalize(S.data_ptr(), m, totals.data_ptr(), G, g, idx.data_ptr(),
                                            dlib.stream_handle()), "dr_shard_finalize")

    build = []
    for g in range(G):
        build.append({"rank": g,
                      "deferred_ms": timed(lambda: DeviceShardOps(True).finalize(DeviceShardOps(True).shard_scan(
                          parts[g])[0], totals, G, g)),
                      "two_pass_ms": timed(lambda: legacy_build(parts[g], g))})
    res[f"build_G{G}"] = {"slowest_rank_deferred_ms": max(b["deferred_ms"] for b in build),
                          "slowest_rank_two_pass_ms": max(b["two_pass_ms"] for b in build), "ranks": build}
    per = []
    for g in range(G):
        ucap, ocap = slice_capacity(tabs[g], N, ts)
        out = torch.empty(max(ocap, 1), dtype=torch.int64, device="cuda")

        def rank_step():
            ops.unif_tile_totals((k0, k1), 0, N, bounds[g], bounds[g + 1])
            U, rng, _ = ops.unif_local((k0, k1), 0, N, agg_all, zmin_all, totals, G, g, ucap, ocap, False)
            ops.shard_match(tabs[g], U, rng, N, out)
        U, rng, st = ops.unif_local((k0, k1), 0, N, agg_all, zmin_all, totals, G, g, ucap, ocap, False)
        a, b, ta, tb = rng.tolist()[:4]
        per.append({"rank": g, "ms": timed(rank_step), "draws": b - a, "tiles_regenerated": tb - ta + 1,
                    "status": int(st.item())})
    slowest = max(p["ms"] for p in per)
    res[f"G{G}"] = {"slowest_rank_ms": slowest, "sum_ms": sum(p["ms"] for p in per), "ranks": per}
    del tabs
    torch.cuda.empty_cache()
print(json.dumps(res))
