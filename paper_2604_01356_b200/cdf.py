"""Cumulative weight tables on the GPU (drop-in for dacresample.cdf).

Mirrors /root/reference/pkg/src/dacresample/cdf.py: ``WeightTable`` (:20-56),
``build_weight_table`` (:59-89) and ``upper_bound_search`` (:92-126), with the
same names, argument meaning and error messages.  The table lives in HBM:
a value array (fp64[M]) plus its index buffer (16-ary search levels, top
guide, table header).  ``build_weight_table`` makes a *deferred* table in one
pass over the weights (``dr_build_table_deferred``): the values are the
in-tile chained sums and the cumulative weights W_j = fl(S_j / T) are formed
where a search compares them (include/drs.h); they are
bit-identical to the two-pass ``dr_build_table``'s W.  ``WeightTable(cum)``
makes a *direct* table holding ``cum`` itself.  ``.cum`` is a lazily mirrored,
read-only host copy kept for reference compatibility.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from ._tensors import is_device_tensor, read_status, status_word, to_device_f64

__all__ = ["WeightTable", "build_weight_table", "build_weight_table_from_log", "upper_bound_search"]


def _raise_build_status(st: int) -> None:
    # priority of the reference's checks (cdf.py:72-84)
    if st & _lib.ST_INVALID_WEIGHT:
        raise ValueError("invalid weight")
    if st & _lib.ST_DEGENERATE:
        raise ValueError("degenerate distribution")
    if st & _lib.ST_ACCUM_OVERFLOW:
        raise ValueError("accumulation overflow")


def _raise_table_status(st: int) -> None:
    # WeightTable.__init__ order (cdf.py:33-40)
    if st & _lib.ST_NONFINITE:
        raise ValueError("invalid weight")
    if st & _lib.ST_DECREASING:
        raise ValueError("cumulative weights must be non-decreasing from >= 0")
    if st & _lib.ST_TOP_NOT_ONE:
        raise ValueError("cumulative weights must end at exactly 1")


def _new_index(m: int) -> torch.Tensor:
    n = int(_lib.lib().dr_index_entries(m))  # levels, top guide, table header: > 0 for every m
    return torch.empty(n, dtype=torch.float64, device=_lib.device())


def _ptr(t) -> int:
    return 0 if t is None else t.data_ptr()


class WeightTable:
    """Immutable cumulative weights of a normalized discrete distribution.

    ``cum[j]`` is the total mass at indices <= j and ``cum[-1]`` is exactly
    1.0 (cdf.py:20-30).  Device-resident; shareable across threads, all
    searches are reentrant.
    """

    __slots__ = ("_W", "_idx", "_host", "_deferred", "_cumdev")

    def __init__(self, cum, *, _built=None):
        self._host = None
        self._cumdev = None
        if _built is not None:
            self._W, self._idx, self._deferred = _built
            return
        self._deferred = False
        if is_device_tensor(cum):
            if cum.ndim != 1 or cum.numel() == 0:
                raise ValueError("empty distribution")
        else:
            a = np.ascontiguousarray(cum, dtype=np.float64)
            if a.ndim != 1 or a.size == 0:
                raise ValueError("empty distribution")
            cum = a
        W, _ = to_device_f64(cum)
        if W.data_ptr() == getattr(cum, "data_ptr", lambda: None)():
            W = W.clone()  # the table must not alias a caller-writable buffer
        L = _lib.lib()
        st = status_word()
        s = _lib.stream_handle()
        _lib.check(L.dr_validate_table(W.data_ptr(), W.numel(), st.data_ptr(), s), "dr_validate_table")
        _raise_table_status(read_status(st))
        idx = _new_index(W.numel())
        _lib.check(L.dr_build_index(W.data_ptr(), W.numel(), _ptr(idx), s), "dr_build_index")
        self._W, self._idx = W, idx

    # -- reference surface -------------------------------------------------
    @property
    def cum(self) -> np.ndarray:
        """Read-only host mirror of W (copied from the device on first use)."""
        if self._host is None:
            h = self.device_cum.cpu().numpy()
            h.flags.writeable = False
            self._host = h
        return self._host

    @property
    def size(self) -> int:
        return self._W.shape[0]

    def __len__(self) -> int:
        return self._W.shape[0]

    def weights(self) -> np.ndarray:
        """Per-index probabilities recovered from the cumulative sums (cdf.py:51-53)."""
        W = self.device_cum
        return torch.diff(W, prepend=W.new_zeros(1)).cpu().numpy()

    def __repr__(self):
        return f"WeightTable(size={self.size})"

    # -- device surface ------------------------------------------------------
    @property
    def device_cum(self) -> torch.Tensor:
        """W on the device (treat as read-only); a deferred table's is formed
        once (``dr_table_materialize``) and kept."""
        if not self._deferred:
            return self._W
        if self._cumdev is None:
            W = torch.empty_like(self._W)
            _lib.check(_lib.lib().dr_table_materialize(self._W.data_ptr(), self._idx.data_ptr(), self.size,
                                                       W.data_ptr(), _lib.stream_handle()), "dr_table_materialize")
            self._cumdev = W
        return self._cumdev

    @property
    def device_values(self) -> torch.Tensor:
        """The value array the searches read (W, or a deferred table's in-tile sums)."""
        return self._W

    @property
    def deferred(self) -> bool:
        return self._deferred

    @property
    def device_index(self) -> torch.Tensor | None:
        return self._idx


def build_weight_table(raw_weights, *, check: bool = True, deferred: bool = True) -> WeightTable:
    """Normalize nonnegative weights into a :class:`WeightTable` (cdf.py:59-89).

    One pass over the weights (``deferred=True``, ``dr_build_table_deferred``):
    validate + chained fp64 scan into in-tile sums, the tile chain, then the
    index levels of W = S / T (``W[M-1] = 1``).  ``deferred=False`` runs the
    two-pass build that stores W itself (``dr_build_table``); both tables have
    the same W and give the same indices.  Raises ``ValueError`` with the
    reference's messages ("empty distribution", "invalid weight", "degenerate
    distribution", "accumulation overflow").  ``check=False`` skips the 4-byte
    status read (and therefore the host synchronisation) for callers that
    validate elsewhere.
    """
    if is_device_tensor(raw_weights):
        if raw_weights.ndim != 1 or raw_weights.numel() == 0:
            raise ValueError("empty distribution")
        w = raw_weights
    else:
        a = np.asarray(raw_weights, dtype=np.float64)
        if a.ndim != 1 or a.size == 0:
            raise ValueError("empty distribution")
        w = a
    w, _ = to_device_f64(w)
    if w.data_ptr() % 16:
        w = w.clone()
    m = w.numel()
    L = _lib.lib()
    W = torch.empty(m, dtype=torch.float64, device=_lib.device())
    idx = _new_index(m)
    st = status_word()
    ws, wsb = _lib.workspace(L.dr_workspace_bytes(_lib.OP_TABLE, m, 0, 0))
    fn = "dr_build_table_deferred" if deferred else "dr_build_table"
    _lib.check(getattr(L, fn)(w.data_ptr(), m, W.data_ptr(), idx.data_ptr(), st.data_ptr(), ws, wsb,
                              _lib.stream_handle()), fn)
    if check:
        _raise_build_status(read_status(st))
    return WeightTable(None, _built=(W, idx, deferred))


def build_weight_table_from_log(log_weights, *, check: bool = True, deferred: bool = True) -> WeightTable:
    """The table of ``exp(log_weights - log_weights.max())`` in one device pipeline.

    The fused weight producer of SURVEY 8(f): the reference's EnGMF field
    shifts its log-weights by the maximum and exponentiates
    (weightgen.py:152-153) before ``build_weight_table`` (cdf.py:59-89); here
    a max reduction and one table pass (``deferred=False``: two) form the
    weights in shared memory (device exp, within 1 ulp of np.exp), so w is
    never written.
    Errors as ``build_weight_table`` (a NaN log-weight is an "invalid weight").
    """
    if is_device_tensor(log_weights):
        if log_weights.ndim != 1 or log_weights.numel() == 0:
            raise ValueError("empty distribution")
        lw = log_weights
    else:
        a = np.asarray(log_weights, dtype=np.float64)
        if a.ndim != 1 or a.size == 0:
            raise ValueError("empty distribution")
        lw = a
    lw, _ = to_device_f64(lw)
    if lw.data_ptr() % 16:
        lw = lw.clone()
    m = lw.numel()
    L = _lib.lib()
    W = torch.empty(m, dtype=torch.float64, device=_lib.device())
    idx = _new_index(m)
    st = status_word()
    ws, wsb = _lib.workspace(L.dr_workspace_bytes(_lib.OP_TABLE, m, 0, 0))
    fn = "dr_build_table_log_deferred" if deferred else "dr_build_table_log"
    _lib.check(getattr(L, fn)(lw.data_ptr(), m, W.data_ptr(), idx.data_ptr(), st.data_ptr(), ws, wsb,
                              _lib.stream_handle()), fn)
    if check:
        _raise_build_status(read_status(st))
    return WeightTable(None, _built=(W, idx, deferred))


def upper_bound_search(table: WeightTable, lo: int, hi: int, x: float, stats=None) -> int:
    """Smallest index j in [lo, hi] with cum[j] >= x (hi if none qualifies).

    cdf.py:92-126; probes are counted on the device when ``stats`` is given.
    """
    lo = int(lo)
    hi = int(hi)
    if lo > hi:
        raise ValueError("empty range")
    if lo < 0 or hi >= table.size:
        raise IndexError("search range outside table")
    out = torch.empty(2, dtype=torch.int64, device=_lib.device())
    _lib.check(
        _lib.lib().dr_lower_bound_range(table.device_cum.data_ptr(), lo, hi, float(x), out.data_ptr(), _lib.stream_handle()),
        "dr_lower_bound_range",
    )
    j, probes = (int(v) for v in out.cpu().tolist())
    if stats is not None:
        stats.probes += probes
    return j
