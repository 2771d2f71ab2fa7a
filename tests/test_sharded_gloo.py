"""Multi-rank logic of the W-sharded table on CPU ranks (gloo), world sizes 2-4.

The collective part of paper_2604_01356_b200.sharded -- the single all-gather
of (T_g, M_g, status_g), the rank-order fold of the shard offsets, error
agreement across ranks, and the U-slice routing that sends every u to
exactly one rank -- runs unchanged; the four device steps are replaced by
an oracle-backed ``ops`` object (test infrastructure).  The result must equal
the oracle's sharded table and its lower bounds.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class Stream:
    def __init__(self, seed):
        from oracle import oracle as orc

        self.key = orc.key_of(seed)
        self.position = 0


class OracleShardOps:
    """CPU stand-in for DeviceShardOps (same four steps, numpy + oracle)."""

    def __init__(self):
        from oracle import oracle as orc

        self.orc = orc

    def device(self):
        return torch.device("cpu")

    def shard_scan(self, w):
        a = w.numpy()
        if a.size == 0:
            return torch.zeros(0, dtype=torch.float64), torch.zeros(1, dtype=torch.float64), torch.zeros(1, dtype=torch.int32)
        S, T = self.orc.chain_scan(a, 33)
        st = 0 if np.all((a >= 0) & np.isfinite(a)) else 1
        if T == 0.0:
            st |= 0x2  # like dr_shard_scan: the LOCAL total is degenerate
        return torch.from_numpy(S), torch.tensor([T], dtype=torch.float64), torch.tensor([st], dtype=torch.int32)

    @staticmethod
    def _fold(totals, g):
        O = 0.0
        for v in totals[:g]:
            O = O + v
        return O

    def finalize(self, S, totals, G, g):
        if S.numel() == 0:
            return S, None
        tv = totals.tolist()
        Og, T = self._fold(tv, g), self._fold(tv, G)
        W = np.minimum((Og + S.numpy()) / T, 1.0)
        if g == G - 1:
            W[-1] = 1.0
        return torch.from_numpy(W), torch.from_numpy(self.orc.build_index(W))

    def tile_size(self):
        return 32 * 8 * 2  # LANES * WARPS * K_UNIF of the device association

    def _spacings(self, key, offset, n):
        return self.orc.neglog(self.orc.uniforms(key[0], key[1], offset, n + 1))

    def unif_tile_totals(self, key, offset, n, t0, t1):
        ts = self.tile_size()
        z = self._spacings(key, offset, n)
        agg, zmin = [], []
        for t in range(t0, t1):
            zt = np.zeros(ts)
            part = z[t * ts:(t + 1) * ts]
            zt[: part.size] = part
            agg.append(self.orc.chain_scan(zt, 2)[1])
            zmin.append(part.min())
        return torch.tensor(agg, dtype=torch.float64), torch.tensor(zmin, dtype=torch.float64)

    def unif_local(self, key, offset, n, agg_all, zmin_all, totals, G, g, ucap, ocap, full):
        ts = self.tile_size()
        # the gathered tile totals are exactly this stream's (all ranks' shares)
        nt = (n + 1 + ts - 1) // ts
        ref, _ = self.unif_tile_totals(key, offset, n, 0, nt)
        assert np.array_equal(agg_all.numpy(), ref.numpy())
        U, _ = self.orc.sorted_uniforms(key[0], key[1], offset, n)
        tv = totals.tolist()
        T = self._fold(tv, G)
        lo = 0 if g == 0 else int(np.searchsorted(U, min(self._fold(tv, g) / T, 1.0), side="right"))
        hi = n if g == G - 1 else int(np.searchsorted(U, min(self._fold(tv, g + 1) / T, 1.0), side="right"))
        st = 0
        if hi - lo > ocap:  # the index window is too small: empty slice, SHARD_CAPACITY
            hi, st = lo, 0x200
        # full-length U window (base 0); the index window starts at the slice
        rng = torch.tensor([lo, hi, 0, nt - 1, 0, lo, 0, 0], dtype=torch.int64)
        return torch.from_numpy(U), rng, torch.tensor([st], dtype=torch.int32)

    def shard_match(self, table, U, rng, n, out):
        if table.W.numel() == 0:
            return out
        a, b = rng.tolist()[:2]
        ob = int(rng[5])
        W = table.W.numpy()
        u = U.numpy()
        for i in range(a, b):
            out[i - ob] = table.start + self.orc.upper_bound(W, 0, W.shape[0] - 1, u[i])
        return out


def _weights(M, bad_rank_slice=None):
    rng = np.random.default_rng(1005)
    w = np.exp(2 * rng.standard_normal(M))
    w[rng.random(M) < 0.05] = 0.0
    if M < 128:
        w[-1] = 1.0
        return w
    off = int(rng.integers(0, M - 64))
    w[off:off + 64] = (w.sum() - w[off:off + 64].sum()) / 3 / 64
    return w


def _worker(rank, world, port, M, N, mode, q):
    import sys
    from pathlib import Path

    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2604_01356_b200 import sharded
        from paper_2604_01356_b200.sharded import build_sharded_table, sharded_dac_sampler

        ops = OracleShardOps()
        w = _weights(M)
        if mode == "zero_shard":  # one shard all zero, the total positive
            w[M * 1 // world: M * 2 // world] = 0.0
        a, b = M * rank // world, M * (rank + 1) // world
        part = w[a:b].copy()
        if mode == "invalid" and rank == world - 1:
            part[3] = -1.0
        if mode == "degenerate":
            part[:] = 0.0
        if mode == "tinycap":  # windows too small: SHARD_CAPACITY, re-run at full size
            sharded.slice_capacity = lambda table, n, tile, g=None: (8, 2)
        try:
            table = build_sharded_table(torch.from_numpy(part), ops=ops)
        except ValueError as e:
            q.put((rank, "error", str(e)))
            return
        comm = "none" if mode == "nocomm" else "allgather"
        out, rng = sharded_dac_sampler(table, N, Stream(2005), ops=ops, gather=True, comm=comm)
        q.put((rank, "ok", (table.W.numpy(), table.start, out.numpy(), rng.tolist(), table.totals.numpy(), w)))
    finally:
        dist.destroy_process_group()


def _run(world, M, N, mode="ok"):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, M, N, mode, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    return sorted(res)


@pytest.mark.parametrize("world,M,mode", [(2, 20011, "ok"), (3, 20011, "ok"), (4, 20011, "ok"),
                                          (3, 20011, "nocomm"), (4, 20011, "zero_shard"), (2, 20011, "tinycap"),
                                          (4, 3, "ok"), (3, 2, "nocomm")])
def test_sharded_table_and_sampler_match_oracle(orc, world, M, mode):
    """World 2-4, both communication modes, an all-zero shard, empty shards
    (M < G) and the capacity re-run: the sharded table equals the oracle's,
    the slices tile [0, N), the gathered indices equal the oracle's DaC."""
    N = 3001
    res = _run(world, M, N, mode)
    assert all(r[1] == "ok" for r in res), res
    w = res[0][2][5]
    W = np.concatenate([r[2][0] for r in res])
    Wo, To, st = orc.build_table_sharded(w, world)
    np.testing.assert_array_equal(W, Wo)
    np.testing.assert_array_equal(res[0][2][4], To)
    k0, k1 = orc.key_of(2005)
    Uo, _ = orc.sorted_uniforms(k0, k1, 0, N)
    expect = orc.match("dac", Wo, Uo)
    ranges = [r[2][3] for r in res]
    # the slices tile [0, N) without overlap, in rank order
    assert ranges[0][0] == 0 and ranges[-1][1] == N
    for r0, r1 in zip(ranges, ranges[1:]):
        assert r0[1] == r1[0]
    for r in res:  # gather=True: every rank holds the full index array
        np.testing.assert_array_equal(r[2][2], expect)


@pytest.mark.parametrize("mode,msg", [("invalid", "invalid weight"), ("degenerate", "degenerate distribution")])
def test_sharded_errors_raise_on_every_rank(mode, msg):
    res = _run(2, 5000, 10, mode)
    assert [r[1] for r in res] == ["error", "error"]
    assert all(r[2] == msg for r in res)
