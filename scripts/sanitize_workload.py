"""A small workload that launches every libdrs kernel once or twice, meant
for compute-sanitizer (memcheck / racecheck / synccheck / initcheck):

    compute-sanitizer --tool memcheck python scripts/sanitize_workload.py

(compute-sanitizer is closed on the GPU pool this was built on, so it has run
only without it; the parity tests are the bounds check there.)

Sizes are small (the sanitizers slow kernels down 10-100x) but cross the
tile, group and index-level edges: table builds (plain, log weights), the
validation / index build of a user table, uniforms and sorted uniforms (Philox
and supplied draws, with a forced collapse), every matcher and sampler (the
fused DaC, the two-pass pipeline, merge tiles with a heavy run, the index
searches), op counts, histogram / chi-square / gather, the batched bank and
the shard steps.  Prints OK at the end; the sanitizer's exit status decides.
"""

import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2604_01356_b200 as drs  # noqa: E402
from paper_2604_01356_b200.sharded import DeviceShardOps, ShardedWeightTable, slice_capacity  # noqa: E402


class Replay:
    def __init__(self, v):
        self.v = np.asarray(v, dtype=np.float64)
        self.draws = 0

    def uniforms(self, k):
        out = self.v[self.draws:self.draws + k]
        self.draws += k
        return out


def main():
    rng = np.random.default_rng(1)
    M = 3 * 8448 + 17
    w = np.exp(3 * rng.standard_normal(M))
    w[rng.random(M) < 0.1] = 0.0
    t = drs.build_weight_table(w)
    drs.build_weight_table_from_log(np.log(w + 1e-300))
    drs.WeightTable(t.cum)  # validation + index build of a user table
    N = 5000
    for mode in ("auto", "merge", "search"):
        drs.dac_sampler(t, N, drs.RngStream(1), mode=mode)
    drs.ccf_sampler(t, N, drs.RngStream(2))
    drs.binary_sampler(t, N, drs.RngStream(3))
    U = drs.sorted_uniforms(drs.RngStream(4), N)
    drs.dac_match(U, t)
    drs.ccf_match(U, t)
    drs.samplers._lower_bounds(t, torch.as_tensor(U, device="cuda"))
    s = drs.OpStats()
    drs.dac_match(U, t, stats=s)
    drs.binary_sampler(t, 200, drs.RngStream(5), stats=drs.OpStats())
    drs.upper_bound_search(t, 0, M - 1, 0.5)
    # a forced collapse through the supplied-draw path (repair)
    d = rng.random(3001)
    d[rng.random(3001) < 0.3] = 1 - 2.0 ** -53
    drs.sorted_uniforms(Replay(d), 3000)
    drs.dac_sampler(t, 3000, Replay(d), mode="search")
    # a heavy run: one weight with most of the mass, N above the split threshold
    wh = np.exp(rng.standard_normal(20000))
    wh[777] = 50 * wh.sum()
    th = drs.build_weight_table(wh)
    drs.ccf_sampler(th, 9000, drs.RngStream(6))
    # extras
    idx = drs.dac_sampler(t, N, drs.RngStream(7), device=True)
    c = drs.histogram(idx, M, device=True)
    drs.chi_square_statistic(c, t, N)
    drs.gather_states(torch.rand(M, 5, dtype=torch.float64, device="cuda"), idx)
    # batched bank (one and two table tiles)
    for Mf, Nf in ((4096, 100), (16384, 256), (9000, 700)):
        B = 20
        wb = np.exp(rng.standard_normal((B, Mf)))
        drs.resample_batched(wb, Nf, [drs.RngStream(8, (b,)) for b in range(B)], return_uniforms=True,
                             return_tables=True)
    # shard steps, G = 2 on one device
    ops = DeviceShardOps()
    G, n = 2, 4000
    parts = [torch.as_tensor(w[M * g // G: M * (g + 1) // G], device="cuda") for g in range(G)]
    scans = [ops.shard_scan(p) for p in parts]
    totals = torch.cat([x[1] for x in scans])
    ts = ops.tile_size()
    nt = (n + 1 + ts - 1) // ts
    key = drs.RngStream(9).key
    agg, zmin = ops.unif_tile_totals(key, 0, n, 0, nt)
    for g in range(G):
        W, ix = ops.finalize(scans[g][0], totals, G, g)
        tab = ShardedWeightTable(W=W, index=ix, totals=totals, sizes=[p.numel() for p in parts], rank=g, world=G,
                                 totals_host=totals.cpu().tolist())
        ucap, ocap = slice_capacity(tab, n, ts)
        Uw, r8, st = ops.unif_local(key, 0, n, agg, zmin, totals, G, g, ucap, ocap, False)
        out = torch.empty(max(ocap, 1), dtype=torch.int64, device="cuda")
        ops.shard_match(tab, Uw, r8, n, out)
    torch.cuda.synchronize()
    print("OK")


if __name__ == "__main__":
    main()
