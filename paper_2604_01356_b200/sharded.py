"""One weight table split in contiguous ranges over the GPUs of a process group.

The multi-GPU mode of the north star (config 5, M = 2^30): rank g of G owns
``w[start_g : start_g + M_g)`` and never holds the rest.

1. ``dr_shard_scan``: local chained scan S and local total T_g (device).
2. ONE all-gather of (T_g, M_g, status_g) -- 24 bytes per rank, NCCL over
   NVLink -- gives every rank all totals, shard sizes and error states.
3. ``dr_shard_finalize``: O_g = T_0 + ... + T_{g-1} and T = O_G folded in
   rank order on every rank, W = min((O_g + S)/T, 1) in place, index built.
   Rank g's lower boundary fl(O_g/T) is bit-identical to rank g-1's last W.
4. Sampling without replicating U.  The tile chain of the n + 1 spacings
    needs every spacing tile's total:
   - ``comm="allgather"``: rank g generates the totals of its 1/G of the
     spacing tiles (``dr_shard_unif_totals``) and ONE all-gather of those
     totals (8 bytes per tile, plus the tiles' spacing minima) gives all;
   - ``comm="none"``: every rank generates all tile totals itself -- no
     collective at all after the table build (the north star's literal
     "no further communication"), at the price of the full Philox + log pass
     on every rank.
   Every rank then folds the identical tile chain, regenerates only the tiles
   holding the u's of its W range (fl(O_g/T), fl(O_{g+1}/T)] plus the tile
   before them (so a repair chain entering the slice is repaired from its
   start), and matches that slice against its shard (``dr_shard_unif_local``,
   ``dr_shard_match``).  U and the indices live in slice-sized windows; the U
   values are bit-identical to ``dr_sorted_uniforms`` on every slice.

The compute steps go through an ``ops`` object (default: the CUDA library)
so that the collective logic can be exercised on CPU ranks with gloo in the
tests, where an oracle-backed ``ops`` stands in for the device.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import torch
import torch.distributed as dist

__all__ = ["ShardedWeightTable", "build_sharded_table", "sharded_dac_sampler", "DeviceShardOps",
           "slice_capacity"]

ST_DEGENERATE = 0x2
ST_SHARD_CAPACITY = 0x200
ST_SHARD_WINDOW = 0x400


class DeviceShardOps:
    """The CUDA implementation of the shard steps (libdrs.so)."""

    def __init__(self, deferred: bool = True):
        from . import _lib

        self._lib = _lib
        # deferred: single-pass shards (16 bytes per entry, no pass after the
        # all-gather); else the two-pass shards holding W itself
        self.deferred = deferred

    def device(self):
        return self._lib.device()

    def shard_scan(self, w: torch.Tensor):
        """(scan, T_g, status): the shard's single pass (dr_shard_scan_deferred:
        in-tile sums, level-1 index entries and tile pairs) or its two-pass local
        chained prefix (dr_shard_scan), and the local total."""
        m = w.numel()
        Tg = torch.zeros(1, dtype=torch.float64, device=w.device)
        st = torch.zeros(1, dtype=torch.int32, device=w.device)
        if m == 0:  # an empty shard owns no weights: total 0, no error of its own
            return _ShardScan(torch.empty(0, dtype=torch.float64, device=w.device), None), Tg, st
        L = self._lib.lib()
        V = torch.empty(m, dtype=torch.float64, device=w.device)
        idx = torch.empty(int(L.dr_index_entries(m)), dtype=torch.float64, device=w.device)
        ws, wsb = self._lib.workspace(L.dr_workspace_bytes(self._lib.OP_TABLE, m, 0, 0))
        if self.deferred:
            self._lib.check(L.dr_shard_scan_deferred(w.data_ptr(), m, V.data_ptr(), idx.data_ptr(), Tg.data_ptr(),
                                                     st.data_ptr(), ws, wsb, self._lib.stream_handle()),
                            "dr_shard_scan_deferred")
        else:
            self._lib.check(L.dr_shard_scan(w.data_ptr(), m, V.data_ptr(), Tg.data_ptr(), st.data_ptr(), ws, wsb,
                                            self._lib.stream_handle()), "dr_shard_scan")
        return _ShardScan(V, idx), Tg, st

    def finalize(self, S, totals: torch.Tensor, G: int, g: int):
        """(values, index) of the shard once the totals are known: the header
        {T, 2, O_g, pin} and the index levels of W (dr_shard_finalize_deferred),
        or W = min((O_g + S) / T, 1) in place and its index (dr_shard_finalize)."""
        if S.numel() == 0:
            return S.V, None
        L = self._lib.lib()
        if self.deferred:
            self._lib.check(L.dr_shard_finalize_deferred(S.numel(), totals.data_ptr(), G, g, S.idx.data_ptr(),
                                                         self._lib.stream_handle()), "dr_shard_finalize_deferred")
        else:
            self._lib.check(L.dr_shard_finalize(S.V.data_ptr(), S.numel(), totals.data_ptr(), G, g,
                                                S.idx.data_ptr(), self._lib.stream_handle()), "dr_shard_finalize")
        return S.V, S.idx

    def materialize(self, V: torch.Tensor, idx: torch.Tensor | None) -> torch.Tensor:
        """The shard's cumulative weights W (dr_table_materialize)."""
        if V.numel() == 0 or idx is None:
            return V
        W = torch.empty_like(V)
        self._lib.check(self._lib.lib().dr_table_materialize(V.data_ptr(), idx.data_ptr(), V.numel(), W.data_ptr(),
                                                             self._lib.stream_handle()), "dr_table_materialize")
        return W

    def tile_size(self) -> int:
        lanes, warps, _, k_unif, _, _ = self._lib.scan_geometry()
        return lanes * warps * k_unif

    def unif_tile_totals(self, key, offset: int, n: int, t0: int, t1: int):
        dev = self.device()
        agg = torch.empty(max(t1 - t0, 1), dtype=torch.float64, device=dev)
        zmin = torch.empty(max(t1 - t0, 1), dtype=torch.float64, device=dev)
        self._lib.check(self._lib.lib().dr_shard_unif_totals(key[0], key[1], offset, n, t0, t1, agg.data_ptr(),
                                                             zmin.data_ptr(), self._lib.stream_handle()),
                        "dr_shard_unif_totals")
        return agg[: t1 - t0], zmin[: t1 - t0]

    def unif_local(self, key, offset: int, n: int, agg_all: torch.Tensor, zmin_all: torch.Tensor,
                   totals: torch.Tensor, G: int, g: int, ucap: int, ocap: int, full: bool):
        """(U window, range8, status) -- see include/drs.h dr_shard_unif_local."""
        L = self._lib.lib()
        dev = self.device()
        U = torch.empty(ucap, dtype=torch.float64, device=dev)
        rng = torch.empty(8, dtype=torch.int64, device=dev)
        st = torch.empty(1, dtype=torch.int32, device=dev)
        ws, wsb = self._lib.workspace(self._lib.workspace_bytes(self._lib.OP_SORTED, n))
        agg_all = agg_all.contiguous()
        zmin_all = zmin_all.contiguous()
        self._lib.check(L.dr_shard_unif_local(key[0], key[1], offset, n, agg_all.data_ptr(), zmin_all.data_ptr(),
                                              zmin_all.numel(), totals.data_ptr(), G, g, U.data_ptr(), ucap, ocap,
                                              int(full), rng.data_ptr(), st.data_ptr(), ws, wsb,
                                              self._lib.stream_handle()),
                        "dr_shard_unif_local")
        return U, rng, st

    def shard_match(self, table: "ShardedWeightTable", U: torch.Tensor, rng: torch.Tensor, n: int,
                    out: torch.Tensor) -> torch.Tensor:
        if table.W.numel() == 0:  # an empty shard is routed no u
            return out
        idx = table.index
        self._lib.check(self._lib.lib().dr_shard_match(
            table.W.data_ptr(), 0 if idx is None else idx.data_ptr(), table.W.numel(), table.start,
            U.data_ptr(), n, rng.data_ptr(), out.data_ptr(), self._lib.stream_handle()), "dr_shard_match")
        return out


class _ShardScan:
    """A shard after its scan: the value array and the index buffer the scan
    wrote into (level 1 and the tile pairs), until finalize completes them."""

    def __init__(self, V: torch.Tensor, idx: torch.Tensor | None):
        self.V, self.idx = V, idx

    def numel(self) -> int:
        return self.V.numel()

    @property
    def device(self):
        return self.V.device


@dataclass
class ShardedWeightTable:
    """This rank's shard of a table spread over a process group."""

    W: torch.Tensor            # the shard's value array (W itself, or a deferred shard's in-tile sums)
    index: torch.Tensor | None  # search index of the shard (its header tells which)
    totals: torch.Tensor       # all shard totals, rank order (device)
    sizes: list[int]           # all shard sizes
    rank: int
    world: int
    group: object = None
    totals_host: list[float] = field(default_factory=list)  # the same totals on the host
    deferred: bool = False     # W holds a deferred shard's values (DeviceShardOps)

    @property
    def cum(self) -> torch.Tensor:
        """The shard's cumulative weights (formed on the device for a deferred shard)."""
        if not self.deferred or self.index is None or self.W.numel() == 0:
            return self.W
        return DeviceShardOps().materialize(self.W, self.index)

    @property
    def start(self) -> int:
        return sum(self.sizes[: self.rank])

    @property
    def size(self) -> int:
        return sum(self.sizes)

    def boundaries(self, g: int | None = None) -> tuple[float, float]:
        """(fl(O_g / T), fl(O_{g+1} / T)): rank g's u range, folded in rank order like the device."""
        g = self.rank if g is None else g
        o, Og, Og1 = 0.0, 0.0, 0.0
        for h, v in enumerate(self.totals_host):
            if h == g:
                Og = o
            o = o + v
            if h == g:
                Og1 = o
        return min(Og / o, 1.0), min(Og1 / o, 1.0)


def slice_capacity(table: ShardedWeightTable, n: int, tile: int, g: int | None = None) -> tuple[int, int]:
    """(U window, index window) sizes for rank g's slice of n sorted uniforms.

    The slice size is Binomial(n, q), q = the rank's share of the mass; the
    index window holds its mean plus 12 standard deviations (a shortfall sets
    SHARD_CAPACITY and the call is re-run at full size), the U window adds
    the partial tiles at both ends, the tile before them and the leading slot.
    """
    lo, hi = table.boundaries(g)
    q = max(0.0, hi - lo)
    if table.world == 1 or q >= 1.0:
        return n + 1, n
    ocap = min(n, int(n * q + 12.0 * math.sqrt(n * q * (1.0 - q)) + 64))
    return min(n + 1, ocap + 3 * tile + 1), ocap


def build_sharded_table(raw_shard, *, group=None, ops=None, deferred: bool = True) -> ShardedWeightTable:
    """Build this rank's shard of one weight table (collective over ``group``).

    ``raw_shard``: this rank's contiguous slice of the raw weights, in rank
    order (it may be empty).  ``deferred``: single-pass shards (the default;
    16 bytes per entry and no pass over the shard after the all-gather) or
    two-pass shards holding W (a table built once and sampled many times).
    Raises the reference's ValueError on every rank
    when any shard is invalid, when the whole table is empty, or when the
    total is degenerate / overflowing -- always after the collective, so no
    rank is left waiting in it.
    """
    ops = ops or DeviceShardOps(deferred)
    G = dist.get_world_size(group)
    g = dist.get_rank(group)
    w = raw_shard if isinstance(raw_shard, torch.Tensor) else torch.as_tensor(raw_shard, dtype=torch.float64)
    w = w.to(device=ops.device(), dtype=torch.float64).contiguous()
    bad_shape = w.ndim != 1
    if bad_shape:
        w = w.reshape(-1)[:0]
    S, Tg, st = ops.shard_scan(w)
    mine = torch.stack([Tg.reshape(()), torch.tensor(float(w.numel()), dtype=torch.float64, device=S.device),
                        (st.reshape(()).to(torch.float64) if not bad_shape
                         else torch.tensor(-1.0, dtype=torch.float64, device=S.device))])
    allv = torch.empty(3 * G, dtype=torch.float64, device=S.device)
    dist.all_gather_into_tensor(allv, mine, group=group)
    allv = allv.reshape(G, 3)
    totals = allv[:, 0].contiguous()
    meta = allv.cpu()
    totals_host = [float(v) for v in meta[:, 0].tolist()]
    sizes = [int(v) for v in meta[:, 1].tolist()]
    stats = [int(v) for v in meta[:, 2].tolist()]
    if any(s < 0 for s in stats) or sum(sizes) == 0:
        raise ValueError("empty distribution")
    # a shard whose weights are all zero is fine when the global total is not:
    # degenerate / overflow are properties of T = O_G, folded in rank order
    # like the device does
    st_glob = 0
    for s in stats:
        st_glob |= s & ~ST_DEGENERATE
    T = 0.0
    for v in totals_host:
        T = T + v
    if T == 0.0:
        st_glob |= ST_DEGENERATE
    if not T < float("inf"):
        st_glob |= 0x4
    from .cdf import _raise_build_status

    _raise_build_status(st_glob)
    W, idx = ops.finalize(S, totals, G, g)
    return ShardedWeightTable(W=W, index=idx, totals=totals, sizes=sizes, rank=g, world=G, group=group,
                              totals_host=totals_host, deferred=bool(getattr(ops, "deferred", False)))


def _key_and_take(stream, k: int):
    """(Philox key, draw offset) of the next k draws; advances the stream."""
    if hasattr(stream, "_take"):
        return stream.key, stream._take(k)
    off = stream.position
    stream.position += k
    return stream.key, off


def _all_tile_totals(ops, key, off, n, nt, G, g, group, comm):
    if comm == "none" or G == 1:
        return ops.unif_tile_totals(key, off, n, 0, nt)
    bounds = [nt * h // G for h in range(G + 1)]
    t0, t1 = bounds[g], bounds[g + 1]
    width = (nt + G - 1) // G
    agg, zmin = ops.unif_tile_totals(key, off, n, t0, t1)
    mine = torch.zeros(2 * width, dtype=torch.float64, device=agg.device)
    mine[width:] = float("inf")
    mine[: t1 - t0] = agg
    mine[width: width + t1 - t0] = zmin
    allv = torch.empty(G * 2 * width, dtype=torch.float64, device=agg.device)
    dist.all_gather_into_tensor(allv, mine, group=group)
    allv = allv.reshape(G, 2 * width)
    agg_all = torch.cat([allv[h, : bounds[h + 1] - bounds[h]] for h in range(G)])
    zmin_all = torch.cat([allv[h, width: width + bounds[h + 1] - bounds[h]] for h in range(G)])
    return agg_all, zmin_all


def sharded_dac_sampler(table: ShardedWeightTable, n: int, stream, *, ops=None, gather: bool = False,
                        comm: str = "allgather", check: bool = True):
    """dac_sampler over a sharded table (samplers.py:262-266 semantics).

    ``stream`` must be identical on all ranks.  ``comm``: "allgather" (rank g
    generates the totals of its 1/G of the spacing tiles, one all-gather of
    those) or "none" (every rank generates all tile totals; no collective).
    Each rank then regenerates only the tiles holding its u's and matches them
    against its shard.  Returns ``(out, range8)``: ``out`` is this rank's
    index window -- ``out[i - range8[5]]`` is the index of u number i for
    ``range8[0] <= i < range8[1]`` -- and ``range8`` the device int64[8] of
    include/drs.h.  ``check`` reads the status (one 4-byte sync) and re-runs
    at full size in the rare cases the windows were too small or a repair
    chain started before them.  ``gather=True`` assembles the full int64[n]
    index array on every rank (all-gather of the slices).
    """
    ops = ops or DeviceShardOps()
    n = int(n)
    if n < 1:
        raise ValueError("n must be >= 1")
    if comm not in ("allgather", "none"):
        raise ValueError(f"unknown comm mode {comm!r}")
    G, g = table.world, table.rank
    ts = ops.tile_size()
    nt = (n + 1 + ts - 1) // ts
    key, off = _key_and_take(stream, n + 1)
    agg_all, zmin_all = _all_tile_totals(ops, key, off, n, nt, G, g, table.group, comm)
    ucap, ocap = slice_capacity(table, n, ts)
    U, rng, st = ops.unif_local(key, off, n, agg_all, zmin_all, table.totals, G, g, ucap, ocap, False)
    out = torch.empty(max(ocap, 1), dtype=torch.int64, device=U.device)
    ops.shard_match(table, U, rng, n, out)
    if check and int(st.item()) & (ST_SHARD_CAPACITY | ST_SHARD_WINDOW):
        U, rng, st = ops.unif_local(key, off, n, agg_all, zmin_all, table.totals, G, g, n + 1, n, True)
        out = torch.empty(n, dtype=torch.int64, device=U.device)
        ops.shard_match(table, U, rng, n, out)
    if gather:
        return _gather_slices(out, rng, n, table.group, G), rng
    return out, rng


def _gather_slices(out: torch.Tensor, rng: torch.Tensor, n: int, group, G: int) -> torch.Tensor:
    """The full index array on every rank: all-gather the ranges, then the
    slices padded to the longest one."""
    rngs = torch.empty(8 * G, dtype=torch.int64, device=rng.device)
    dist.all_gather_into_tensor(rngs, rng.contiguous(), group=group)
    r = rngs.reshape(G, 8).cpu().tolist()
    width = max(1, max(x[1] - x[0] for x in r))
    mine = torch.empty(width, dtype=torch.int64, device=out.device)
    k = min(width, out.numel())
    mine[:k] = out[:k]
    allv = torch.empty(G * width, dtype=torch.int64, device=out.device)
    dist.all_gather_into_tensor(allv, mine, group=group)
    allv = allv.reshape(G, width)
    full = torch.full((n,), -1, dtype=torch.int64, device=out.device)
    for h in range(G):
        i0, i1 = r[h][0], r[h][1]
        if i1 > i0:
            full[i0:i1] = allv[h, : i1 - i0]
    return full
