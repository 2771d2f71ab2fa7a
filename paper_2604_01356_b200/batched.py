"""Many independent filters resampled in one launch (config 4).

The reference resamples a bank of filters with a Python loop: per filter
``build_weight_table(w_f)`` (cdf.py:59-89) then ``dac_sampler(table, n,
stream_f)`` (samplers.py:262-266).  ``resample_batched`` gives the identical
per-filter result -- the same W association, the same sorted uniforms for
the same stream, the same lower bounds -- from one ``dr_resample_batched``
launch with one CTA per filter.  Across GPUs the filters shard by rank with
no collective (``shard_filters``).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from ._tensors import finish_host, host_result_i64, is_device_tensor, read_status, status_word, to_device_f64
from .cdf import _raise_build_status
from .randkit import RngStream

__all__ = ["resample_batched", "stream_keys", "shard_filters", "BatchedStreams"]


def stream_keys(streams, n: int) -> torch.Tensor:
    """(B, 3) uint64 [k0, k1, draw offset] for a sequence of RngStream, advancing
    each by n + 1 draws exactly as ``sorted_uniforms`` would."""
    rows = []
    for s in streams:
        if not isinstance(s, RngStream):
            raise TypeError("resample_batched needs RngStream streams (Philox keys)")
        off = s._take(int(n) + 1) if n > 0 else s.position
        rows.append((s.key[0], s.key[1], off))
    a = np.array(rows, dtype=np.uint64).reshape(-1, 3)
    return torch.from_numpy(a.view(np.int64)).to(_lib.device())


class BatchedStreams:
    """B Philox streams whose draw positions live on the device.

    Row b of ``keys`` is (k0, k1, position) of ``RngStream(seed, spawn_key_of(b))``.
    ``resample_batched`` reads the positions on the device and advances
    them by n + 1 there, so a batched call can be captured once in a CUDA
    graph and replayed with fresh draws (the loop of a filter bank).
    """

    __slots__ = ("keys",)

    def __init__(self, streams):
        streams = list(streams)
        rows = [(s.key[0], s.key[1], s.position) for s in streams]
        a = np.array(rows, dtype=np.uint64).reshape(-1, 3)
        self.keys = torch.from_numpy(a.view(np.int64)).to(_lib.device())

    def __len__(self) -> int:
        return int(self.keys.shape[0])

    def positions(self) -> np.ndarray:
        return self.keys[:, 2].cpu().numpy().view(np.uint64)


def resample_batched(raw_weights, n: int, streams, *, return_uniforms: bool = False,
                     return_tables: bool = False, check: bool = True, device: bool = False):
    """Resample B filters of M_f raw weights each, n draws per filter.

    ``raw_weights``: (B, M_f) array-like or CUDA tensor (unnormalised, >= 0).
    ``streams``: B RngStreams (each advanced by n + 1 draws on the host),
    a :class:`BatchedStreams` (positions advanced on the device), or a (B, 3)
    uint64 CUDA tensor of [k0, k1, offset] (not advanced).  Returns int64 indices (B, n);
    with ``return_uniforms`` / ``return_tables`` also U (B, n) / W (B, M_f).
    Errors are raised with ``build_weight_table``'s messages when any filter
    is invalid.
    """
    host = not is_device_tensor(raw_weights)
    w, _ = to_device_f64(raw_weights)
    if w.ndim != 2 or w.shape[1] == 0:
        raise ValueError("raw_weights must be (B, M_f) with M_f >= 1")
    B, Mf = int(w.shape[0]), int(w.shape[1])
    n = int(n)
    if n < 0:
        raise ValueError("n must be >= 0")
    advance = 0
    if isinstance(streams, BatchedStreams):
        if len(streams) != B:
            raise ValueError("need one stream per filter")
        keys, advance = streams.keys, 1
    elif isinstance(streams, torch.Tensor):
        keys = streams.to(_lib.device()).contiguous()
    else:
        streams = list(streams)
        if len(streams) != B:
            raise ValueError("need one stream per filter")
        keys = stream_keys(streams, n)
    dev = _lib.device()
    to_host = host and not device
    out = (host_result_i64(B * n).view(B, n) if to_host
           else torch.empty((B, n), dtype=torch.int64, device=dev))
    U = torch.empty((B, n), dtype=torch.float64, device=dev) if return_uniforms else None
    W = torch.empty((B, Mf), dtype=torch.float64, device=dev) if return_tables else None
    st = status_word()
    rc = _lib.lib().dr_resample_batched(
        w.data_ptr(), B, Mf, n, keys.data_ptr(), advance, 0 if W is None else W.data_ptr(),
        0 if U is None else U.data_ptr(), out.data_ptr(), st.data_ptr(), _lib.stream_handle(),
    )
    _lib.check(rc, "dr_resample_batched")
    if check:
        _raise_build_status(read_status(st))
    res = [out]
    if return_uniforms:
        res.append(U)
    if return_tables:
        res.append(W)
    if to_host:
        res = [finish_host(out)] + [r.cpu().numpy() for r in res[1:]]
    return res[0] if len(res) == 1 else tuple(res)


def shard_filters(B: int, rank: int, world: int) -> slice:
    """Contiguous filter range of one rank (no collective needed)."""
    return slice(B * rank // world, B * (rank + 1) // world)
