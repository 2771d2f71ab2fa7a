"""One weight table split in contiguous ranges over the GPUs of a process group.

The multi-GPU mode of the north star (config 5, M = 2^30): rank g of G owns
``w[start_g : start_g + M_g)`` and never holds the rest.

1. ``dr_shard_scan``: local chained scan S and local total T_g (device).
2. ONE all-gather of (T_g, M_g, status_g) -- 24 bytes per rank, NCCL over
   NVLink -- gives every rank all totals, shard sizes and error states.
3. ``dr_shard_finalize``: O_g = T_0 + ... + T_{g-1} and T = O_G folded in
   rank order on every rank, W = min((O_g + S)/T, 1) in place, index built.
   Rank g's lower boundary fl(O_g/T) is bit-identical to rank g-1's last W.
4. Sampling: every rank regenerates the same sorted U (same stream), finds
   its slice (fl(O_g/T), fl(O_{g+1}/T)] on the device and matches only that
   slice against its shard -- no further communication.

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

    def sorted_uniforms(self, stream, n: int) -> torch.Tensor:
        from .randkit import sorted_uniforms_device

        return sorted_uniforms_device(stream, n)

    def shard_range(self, U: torch.Tensor, totals: torch.Tensor, G: int, g: int) -> torch.Tensor:
        rng = torch.empty(2, dtype=torch.int64, device=U.device)
        self._lib.check(self._lib.lib().dr_shard_range(U.data_ptr(), U.numel(), totals.data_ptr(), G, g,
                                                       rng.data_ptr(), self._lib.stream_handle()),
                        "dr_shard_range")
        return rng

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


def sharded_dac_sampler(table: ShardedWeightTable, n: int, stream, *, ops=None, gather: bool = False):
    """dac_sampler over a sharded table (samplers.py:262-266 semantics).

    Every rank draws the same sorted U from ``stream`` (which must be
    identical on all ranks) and fills the entries of its own slice.  Returns
    ``(out, range)``: ``out`` int64[n] with this rank's slice filled (-1
    elsewhere) and ``range`` = (i0, i1) on the device.  ``gather=True``
    all-reduces (max) so every rank holds the full index array.
    """
    ops = ops or DeviceShardOps()
    U = ops.sorted_uniforms(stream, int(n))
    rng = ops.shard_range(U, table.totals, table.world, table.rank)
    out = ops.shard_match(table, U, rng)
    if gather:
        dist.all_reduce(out, op=dist.ReduceOp.MAX, group=table.group)
    return out, rng
