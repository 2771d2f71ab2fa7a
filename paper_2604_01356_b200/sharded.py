"""One weight table split in contiguous ranges over the GPUs of a process group.

The multi-GPU mode of the north star (config 5, M = 2^30): rank g of G owns
``w[start_g : start_g + M_g)`` and never holds the rest.

1. ``dr_shard_scan``: local chained scan S and local total T_g (device).
2. ONE all-gather of (T_g, M_g, status_g) -- 24 bytes per rank, NCCL over
   NVLink -- gives every rank all totals, shard sizes and error states.
3. ``dr_shard_finalize``: O_g = T_0 + ... + T_{g-1} and T = O_G folded in
   rank order on every rank, W = min((O_g + S)/T, 1) in place, index built.
   Rank g's lower boundary fl(O_g/T) is bit-identical to rank g-1's last W.
4. Sampling without replicating U: rank g generates the totals of its 1/G of
   the spacing tiles (``dr_shard_unif_totals``); ONE all-gather of those
   totals (8 bytes per tile, plus the tiles' spacing minima); every rank folds
   the identical tile chain, regenerates only the tiles holding the u's of its
   W range (fl(O_g/T), fl(O_{g+1}/T)] and matches that slice against its
   shard (``dr_shard_unif_local``, ``dr_shard_match``).  The U values are
   bit-identical to ``dr_sorted_uniforms`` on every slice.

The compute steps go through an ``ops`` object (default: the CUDA library)
so that the collective logic can be exercised on CPU ranks with gloo in the
tests, where an oracle-backed ``ops`` stands in for the device.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist

__all__ = ["ShardedWeightTable", "build_sharded_table", "sharded_dac_sampler", "DeviceShardOps"]


class DeviceShardOps:
    """The CUDA implementation of the four shard steps (libdrs.so)."""

    def __init__(self):
        from . import _lib

        self._lib = _lib

    def device(self):
        return self._lib.device()

    def shard_scan(self, w: torch.Tensor):
        L = self._lib.lib()
        m = w.numel()
        S = torch.empty(m, dtype=torch.float64, device=w.device)
        Tg = torch.empty(1, dtype=torch.float64, device=w.device)
        st = torch.zeros(1, dtype=torch.int32, device=w.device)
        ws, wsb = self._lib.workspace(L.dr_workspace_bytes(self._lib.OP_TABLE, m, 0, 0))
        self._lib.check(L.dr_shard_scan(w.data_ptr(), m, S.data_ptr(), Tg.data_ptr(), st.data_ptr(), ws, wsb,
                                        self._lib.stream_handle()), "dr_shard_scan")
        return S, Tg, st

    def finalize(self, S: torch.Tensor, totals: torch.Tensor, G: int, g: int):
        L = self._lib.lib()
        n = int(L.dr_index_entries(S.numel()))
        idx = torch.empty(n, dtype=torch.float64, device=S.device) if n else None
        self._lib.check(L.dr_shard_finalize(S.data_ptr(), S.numel(), totals.data_ptr(), G, g,
                                            0 if idx is None else idx.data_ptr(), self._lib.stream_handle()),
                        "dr_shard_finalize")
        return S, idx

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
                   totals: torch.Tensor, G: int, g: int):
        L = self._lib.lib()
        dev = self.device()
        U = torch.empty(n, dtype=torch.float64, device=dev)
        rng = torch.zeros(4, dtype=torch.int64, device=dev)
        st = torch.zeros(1, dtype=torch.int32, device=dev)
        ws, wsb = self._lib.workspace(self._lib.workspace_bytes(self._lib.OP_SORTED, n))
        agg_all = agg_all.contiguous()
        zmin_all = zmin_all.contiguous()
        self._lib.check(L.dr_shard_unif_local(key[0], key[1], offset, n, agg_all.data_ptr(), zmin_all.data_ptr(),
                                              zmin_all.numel(), totals.data_ptr(), G, g, U.data_ptr(),
                                              rng.data_ptr(), st.data_ptr(), ws, wsb, self._lib.stream_handle()),
                        "dr_shard_unif_local")
        return U, rng

    def shard_match(self, table: "ShardedWeightTable", U: torch.Tensor, rng: torch.Tensor) -> torch.Tensor:
        out = torch.full((U.numel(),), -1, dtype=torch.int64, device=U.device)
        idx = table.index
        self._lib.check(self._lib.lib().dr_shard_match(
            table.W.data_ptr(), 0 if idx is None else idx.data_ptr(), table.W.numel(), table.start,
            U.data_ptr(), U.numel(), rng.data_ptr(), out.data_ptr(), self._lib.stream_handle()), "dr_shard_match")
        return out


@dataclass
class ShardedWeightTable:
    """This rank's shard of a table spread over a process group."""

    W: torch.Tensor            # normalised cumulative weights of the shard
    index: torch.Tensor | None  # search index of the shard
    totals: torch.Tensor       # all shard totals, rank order (device)
    sizes: list[int]           # all shard sizes
    rank: int
    world: int
    group: object = None

    @property
    def start(self) -> int:
        return sum(self.sizes[: self.rank])

    @property
    def size(self) -> int:
        return sum(self.sizes)


def _raise_status(sts) -> None:
    from .cdf import _raise_build_status

    st = 0
    for s in sts:
        st |= int(s)
    _raise_build_status(st)


def build_sharded_table(raw_shard, *, group=None, ops=None) -> ShardedWeightTable:
    """Build this rank's shard of one weight table (collective over ``group``).

    ``raw_shard``: this rank's contiguous slice of the raw weights, in rank
    order.  Raises the reference's ValueError on every rank when any shard is
    invalid or the total is degenerate/overflowing.
    """
    ops = ops or DeviceShardOps()
    G = dist.get_world_size(group)
    g = dist.get_rank(group)
    w = raw_shard if isinstance(raw_shard, torch.Tensor) else torch.as_tensor(raw_shard, dtype=torch.float64)
    w = w.to(device=ops.device(), dtype=torch.float64).contiguous()
    if w.ndim != 1 or w.numel() == 0:
        raise ValueError("empty distribution")
    S, Tg, st = ops.shard_scan(w)
    mine = torch.stack([Tg.reshape(()), torch.tensor(float(w.numel()), dtype=torch.float64, device=S.device),
                        st.reshape(()).to(torch.float64)])
    allv = torch.empty(3 * G, dtype=torch.float64, device=S.device)
    dist.all_gather_into_tensor(allv, mine, group=group)
    allv = allv.reshape(G, 3)
    totals = allv[:, 0].contiguous()
    meta = allv[:, 1:].cpu()
    sizes = [int(v) for v in meta[:, 0].tolist()]
    stats = [int(v) for v in meta[:, 1].tolist()]
    W, idx = ops.finalize(S, totals, G, g)
    # degenerate / overflow are properties of the global total T = O_G,
    # folded in rank order like the device does
    st_glob = list(stats)
    T = 0.0
    for v in totals.cpu().tolist():
        T = T + v
    if T == 0.0:
        st_glob.append(0x2)
    if not T < float("inf"):
        st_glob.append(0x4)
    _raise_status(st_glob)
    return ShardedWeightTable(W=W, index=idx, totals=totals, sizes=sizes, rank=g, world=G, group=group)


def _key_and_take(stream, k: int):
    """(Philox key, draw offset) of the next k draws; advances the stream."""
    if hasattr(stream, "_take"):
        return stream.key, stream._take(k)
    off = stream.position
    stream.position += k
    return stream.key, off


def sharded_dac_sampler(table: ShardedWeightTable, n: int, stream, *, ops=None, gather: bool = False):
    """dac_sampler over a sharded table (samplers.py:262-266 semantics).

    ``stream`` must be identical on all ranks.  Rank g generates the totals
    of its 1/G of the spacing tiles; one all-gather of those totals; then
    each rank regenerates only the tiles holding its u's and matches them
    against its shard.  Returns ``(out, range)``: ``out`` int64[n] with this
    rank's slice filled (-1 elsewhere) and ``range`` = (i0, i1, first tile,
    last tile) on the device.  ``gather=True`` all-reduces (max) so every
    rank holds the full index array.
    """
    ops = ops or DeviceShardOps()
    n = int(n)
    if n < 1:
        raise ValueError("n must be >= 1")
    G, g = table.world, table.rank
    ts = ops.tile_size()
    nt = (n + 1 + ts - 1) // ts
    bounds = [nt * h // G for h in range(G + 1)]
    t0, t1 = bounds[g], bounds[g + 1]
    width = (nt + G - 1) // G
    key, off = _key_and_take(stream, n + 1)
    agg, zmin = ops.unif_tile_totals(key, off, n, t0, t1)
    mine = torch.zeros(2 * width, dtype=torch.float64, device=agg.device)
    mine[width:] = float("inf")
    mine[: t1 - t0] = agg
    mine[width: width + t1 - t0] = zmin
    allv = torch.empty(G * 2 * width, dtype=torch.float64, device=agg.device)
    dist.all_gather_into_tensor(allv, mine, group=table.group)
    allv = allv.reshape(G, 2 * width)
    agg_all = torch.cat([allv[h, : bounds[h + 1] - bounds[h]] for h in range(G)])
    zmin_all = torch.cat([allv[h, width: width + bounds[h + 1] - bounds[h]] for h in range(G)])
    U, rng = ops.unif_local(key, off, n, agg_all, zmin_all, table.totals, G, g)
    out = ops.shard_match(table, U, rng)
    if gather:
        dist.all_reduce(out, op=dist.ReduceOp.MAX, group=table.group)
    return out, rng
