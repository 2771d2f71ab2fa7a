"""The three multinomial samplers on the GPU (drop-in for dacresample.samplers).

Mirrors /root/reference/pkg/src/dacresample/samplers.py: matchers
``ccf_match`` (:162-188) and ``dac_match`` (:191-210), samplers
``binary_sampler`` (:238-252), ``ccf_sampler`` (:255-259), ``dac_sampler``
(:262-266), ``linear_oracle`` (:49-66), ``OpStats`` (:40-46) and
``warm_kernels`` (:149-156).  Same names, arguments, return dtype (int64,
0-based) and error messages.

Host inputs (lists, numpy) give numpy results, CUDA-tensor inputs give CUDA
tensors; samplers return numpy unless ``device=True``.  Every index is the
unique lower bound ``min{j : W[j] >= u}`` computed on the device -- the
samplers differ in search strategy only, exactly as in the reference.
``stats=`` (an :class:`OpStats`) receives the reference's instrumented
operation counts -- comparisons, probes, max_depth of the CPU algorithms
(samplers.py:178-188, 213-232, 249-252) -- computed exactly on the device
from the table, the uniforms and the indices (``dr_op_counts``).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._tensors import (
    empty_i64,
    finish_host,
    host_result_i64,
    is_device_tensor,
    read_status,
    status_word,
    to_device_f64,
)
from .cdf import WeightTable
from .randkit import DeviceRngStream, RngStream, sorted_uniforms_device

__all__ = [
    "OpStats",
    "linear_oracle",
    "binary_sampler",
    "ccf_match",
    "ccf_sampler",
    "dac_match",
    "dac_sampler",
    "warm_kernels",
]


@dataclass
class OpStats:
    """Operation tallies for verifying complexity claims without a clock."""

    comparisons: int = 0  # weight-vs-uniform comparisons in linear scans
    probes: int = 0       # bisection midpoint evaluations
    max_depth: int = 0    # deepest divide-and-conquer scope nesting


_OP_KIND = {"dac": 0, "ccf": 1, "binary": 2}


def _op_counts(kind: str, table: WeightTable, ud: torch.Tensor, out: torch.Tensor, stats) -> None:
    """Add the reference's instrumented operation counts for this match to
    ``stats`` (samplers.py:178-188, 213-232, 249-252): computed exactly on the
    device from W, the uniforms and the lower bounds (``dr_op_counts``)."""
    n = ud.numel()
    counts = torch.zeros(3, dtype=torch.int64, device=_lib.device())
    if n:
        _lib.check(_lib.lib().dr_op_counts(_OP_KIND[kind], table.device_cum.data_ptr(), table.size, ud.data_ptr(),
                                           n, out.data_ptr(), counts.data_ptr(), _lib.stream_handle()),
                   "dr_op_counts")
    c, p, d = (int(v) for v in counts.cpu().tolist())
    stats.comparisons += c
    stats.probes += p
    if d > stats.max_depth:
        stats.max_depth = d


def _lower_bounds(table: WeightTable, u: torch.Tensor) -> torch.Tensor:
    out = empty_i64(u.numel())
    if u.numel():
        _lib.check(
            _lib.lib().dr_match_binary(
                table.device_values.data_ptr(), _ptr(table.device_index), table.size,
                u.data_ptr(), u.numel(), out.data_ptr(), _lib.stream_handle(),
            ),
            "dr_match_binary",
        )
    return out


def _ptr(t) -> int:
    return 0 if t is None else t.data_ptr()


def linear_oracle(table: WeightTable, u: float, stats=None) -> int:
    """Reference inverse CDF: first j with cum[j] >= u (samplers.py:49-66).

    The answer is the same lower bound as every sampler; the comparison
    count of the reference's linear scan is j + 1.
    """
    u = float(u)
    if not 0.0 < u <= 1.0:
        raise ValueError("u must lie in (0, 1]")
    x = torch.full((1,), u, dtype=torch.float64, device=_lib.device())
    j = int(_lower_bounds(table, x).item())
    if stats is not None:
        stats.comparisons += j + 1
    return j


def _check_sorted_open(u: torch.Tensor) -> None:
    """samplers.py:69-75 on the device; raises with the reference's messages."""
    if u.numel() == 0:
        return
    st = status_word()
    _lib.check(_lib.lib().dr_check_sorted_open(u.data_ptr(), u.numel(), st.data_ptr(), _lib.stream_handle()),
               "dr_check_sorted_open")
    s = read_status(st)
    if s & _lib.ST_OUT_OF_SUPPORT:
        raise ValueError("uniforms must lie in (0, 1]")
    if s & _lib.ST_NOT_SORTED:
        raise ValueError("input not sorted")


def _match(kind: str, u, table: WeightTable, check: bool, mode: str = "auto", stats=None):
    host = not is_device_tensor(u)
    ud, _ = to_device_f64(u)
    if ud.ndim != 1:
        ud = ud.reshape(-1)
    if check:
        _check_sorted_open(ud)
    n = ud.numel()
    out = host_result_i64(n) if host else empty_i64(n)
    if n:
        L = _lib.lib()
        s = _lib.stream_handle()
        W = table.device_values
        if kind == "ccf":
            rc = L.dr_match_ccf(W.data_ptr(), _ptr(table.device_index), table.size, ud.data_ptr(), n,
                                out.data_ptr(), s)
        else:
            rc = L.dr_match_dac(W.data_ptr(), _ptr(table.device_index), table.size, ud.data_ptr(), n,
                                out.data_ptr(), _lib.DAC_MODES[mode], s)
        _lib.check(rc, f"dr_match_{kind}")
    if stats is not None:
        _op_counts(kind, table, ud, out, stats)
    return finish_host(out) if host else out


def ccf_match(u, table: WeightTable, stats: OpStats | None = None, check: bool = True):
    """Match sorted uniforms against the table by a streaming merge (samplers.py:162-188).

    The table is read once, tile by tile (TMA bulk copies into shared
    memory); each tile merges with the slice of u that lands in it.
    """
    return _match("ccf", u, table, check, stats=stats)


def dac_match(u, table: WeightTable, stats: OpStats | None = None, check: bool = True,
              *, mode: str = "auto"):
    """Match sorted uniforms by divide and conquer (samplers.py:191-210).

    ``mode``: "merge" splits u by table tiles and merges each slice (reads
    all of W); "search" splits by index blocks and bisects per u (reads
    O(N log(M/N)) lines); "auto" picks merge when M <= 11 N (the measured crossover).
    """
    if mode not in _lib.DAC_MODES:
        raise ValueError(f"unknown mode {mode!r}")
    return _match("dac", u, table, check, mode, stats=stats)


def _stream_args(stream, n_draws):
    """(k0, k1, offset, offset_dev pointer) for a Philox stream, advancing host streams."""
    if isinstance(stream, DeviceRngStream):
        return stream.key[0], stream.key[1], 0, stream.offset_tensor.data_ptr()
    off = stream._take(n_draws)
    return stream.key[0], stream.key[1], off, 0


def binary_sampler(table: WeightTable, n: int, stream, stats: OpStats | None = None,
                   *, device: bool = False, out=None):
    """n independent draws, each by a full-range search; draw order kept (samplers.py:238-252)."""
    n = int(n)
    if n < 0:
        raise ValueError("negative dimensions are not allowed")
    if out is not None:
        _check_out(out, n, torch.int64, "out")
    if stats is not None:
        # instrumented: the draws are materialised so their probes can be counted
        res = empty_i64(0)
        if n:
            us = _draw_uniforms(stream, n)
            res = _lower_bounds(table, us)
            _op_counts("binary", table, us, res, stats)
        if out is not None:
            out[:n].copy_(res)
            res = out
        return res if device else res.cpu().numpy()
    to_host = out is None and not device
    if out is None:
        out = empty_i64(n) if device else host_result_i64(n)
    if n:
        W = table.device_values
        if isinstance(stream, (RngStream, DeviceRngStream)):
            k0, k1, off, offd = _stream_args(stream, n)
            rc = _lib.lib().dr_sample_binary_dev(W.data_ptr(), _ptr(table.device_index), table.size,
                                                 k0, k1, off, offd, n, out.data_ptr(), _lib.stream_handle())
            _lib.check(rc, "dr_sample_binary_dev")
        else:
            us, _ = to_device_f64(stream.uniforms(n))
            res = _lower_bounds(table, us)
            if res is not out:
                out.copy_(res)
    if to_host:
        return finish_host(out)
    return out if device else out.cpu().numpy()


# Per-(device, stream) scratch.  Buffers are never freed while the process
# runs: a superseded (smaller) scratch U may still be referenced by a CUDA
# graph captured earlier, so it is kept alive in _retired.
_status_cache: dict[tuple[int, int], torch.Tensor] = {}
_scratch_u: dict[tuple[int, int], torch.Tensor] = {}
_retired: list[torch.Tensor] = []


def _status_buf(s: int) -> torch.Tensor:
    """A per-(device, stream) status word the kernels overwrite (no per-call zeroing)."""
    key = (torch.cuda.current_device(), s)
    t = _status_cache.get(key)
    if t is None:
        t = torch.empty(1, dtype=torch.int32, device=_lib.device())
        _status_cache[key] = t
    return t


def _scratch_uniforms(n: int, s: int) -> torch.Tensor:
    """Per-(device, stream) device scratch for U when the caller does not ask
    for it (stream-ordered reuse is safe: every use is on the same stream)."""
    key = (torch.cuda.current_device(), s)
    t = _scratch_u.get(key)
    if t is None or t.numel() < n:
        if t is not None:
            _retired.append(t)
        t = torch.empty(max(n, 1024), dtype=torch.float64, device=_lib.device())
        _scratch_u[key] = t
    return t


def _check_out(buf, n: int, dtype: torch.dtype, name: str) -> None:
    """A caller-supplied output buffer must be a contiguous tensor of the
    right dtype and length, on the current device or device-accessible
    pinned host memory; the kernels write it directly."""
    if not isinstance(buf, torch.Tensor):
        raise TypeError(f"{name} must be a torch.Tensor")
    if buf.dtype != dtype:
        raise ValueError(f"{name} must have dtype {dtype}, got {buf.dtype}")
    if not buf.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if buf.numel() < n:
        raise ValueError(f"{name} holds {buf.numel()} elements, {n} needed")
    if buf.is_cuda:
        if buf.device.index != torch.cuda.current_device():
            raise ValueError(f"{name} is on {buf.device}, the call runs on cuda:{torch.cuda.current_device()}")
    elif not (buf.is_pinned() and (buf.numel() == 0 or _lib.device_accessible(buf.data_ptr()))):
        raise ValueError(f"{name} must be a CUDA tensor or pinned (device-accessible) host memory")


def _draw_uniforms(stream, n: int) -> torch.Tensor:
    """The next n uniforms of a stream, on the device (the stream advances by n)."""
    if isinstance(stream, RngStream):
        return stream.uniforms_device(n)
    if isinstance(stream, DeviceRngStream):
        pos = stream.position
        u = torch.empty(n, dtype=torch.float64, device=_lib.device())
        _lib.check(_lib.lib().dr_uniforms(stream.key[0], stream.key[1], pos, n, u.data_ptr(), _lib.stream_handle()),
                   "dr_uniforms")
        stream.offset_tensor += n
        return u
    return to_device_f64(stream.uniforms(n))[0]


# The per-call host path of the common call (a host RngStream, no out= /
# uniforms_out= / stats=): the per-(device, stream, n) scratch pointers are
# looked up once, and one call into the CPython extension _drshost launches
# dr_sample_dac / dr_sample_ccf and, for a host result, synchronises the
# stream (drs_host.c).  Without the extension the ctypes path below runs the
# same kernels.
try:
    from . import _drshost as _hc
except ImportError:  # not built: the ctypes path
    _hc = None
_hc_bound = False
_plans: dict[tuple[int, int, int], tuple[int, int, int, int]] = {}
_raw_stream = _lib._raw_stream


def _fast_sorted(kind: str, table: WeightTable, n: int, stream: RngStream, device: bool, mode: str):
    global _hc_bound
    dev = torch.cuda.current_device()
    s = _raw_stream(dev)
    plan = _plans.get((dev, s, n))
    if plan is None:
        L = _lib.lib()
        if not _hc_bound:
            addr = lambda f: ctypes.cast(f, ctypes.c_void_p).value  # noqa: E731
            _hc.bind(addr(L.dr_sample_dac), addr(L.dr_sample_dac_sync), addr(L.dr_sample_ccf),
                     addr(L.dr_stream_synchronize))
            _hc_bound = True
        ws, wsb = _lib.workspace(_lib.workspace_bytes(_lib.OP_SORTED, n), s)
        # buffers superseded later stay allocated (_retired / _lib._ws_retired), so a plan stays valid
        plan = (_scratch_uniforms(n, s).data_ptr(), _status_buf(s).data_ptr(), ws, wsb)
        _plans[(dev, s, n)] = plan
    k0, k1 = stream._key
    off = stream._take(n + 1)
    out = empty_i64(n) if device else host_result_i64(n)
    idx = table._idx
    rc = _hc.sorted_sample(0 if kind == "dac" else 1, table._W.data_ptr(), 0 if idx is None else idx.data_ptr(),
                           table.size, k0, k1, off, n, plan[0], out.data_ptr(), plan[1], _lib.DAC_MODES[mode],
                           plan[2], plan[3], s, 0 if device else 1)
    if rc:
        _lib.check(rc, f"dr_sample_{kind}")
    return out if device else out.numpy()


def _sorted_sampler(kind, table, n, stream, stats, device, mode="auto", out=None, U=None):
    if _hc is not None and out is None and U is None and stats is None and type(stream) is RngStream:
        n = int(n)
        if n > 0:
            return _fast_sorted(kind, table, n, stream, device, mode)
    n = int(n)
    if n < 0:
        raise ValueError("n must be >= 0")
    if out is not None:
        _check_out(out, n, torch.int64, "out")
    if U is not None:
        _check_out(U, n, torch.float64, "uniforms_out")
    if n == 0 or stats is not None or (kind == "ccf" and not isinstance(stream, (RngStream, DeviceRngStream))):
        if isinstance(stream, DeviceRngStream):  # the instrumented path draws from the host position
            pos = stream.position
            hs = RngStream(stream.seed, stream._spawn_key)
            hs._take(pos)
            Us = sorted_uniforms_device(hs, n)
            stream.offset_tensor += n + 1 if n else 0
        else:
            Us = sorted_uniforms_device(stream, n)
        res = _match(kind, Us, table, check=False, mode=mode, stats=stats)
        if U is not None and n:
            U[:n].copy_(Us)
        if out is not None:
            if n:
                out[:n].copy_(res)
            res = out
        return res if device else res.cpu().numpy()
    L = _lib.lib()
    s = _lib.stream_handle()
    to_host = out is None and not device
    if out is None:
        out = empty_i64(n) if device else host_result_i64(n)
    U = _scratch_uniforms(n, s) if U is None else U
    st = _status_buf(s)
    ws, wsb = _lib.workspace(_lib.workspace_bytes(_lib.OP_SORTED, n), s)
    W = table.device_values
    if not isinstance(stream, (RngStream, DeviceRngStream)):
        # duck-typed host stream: its n+1 uniforms feed the same fused kernel
        raw, _ = to_device_f64(stream.uniforms(n + 1))
        rc = L.dr_sample_dac_from(W.data_ptr(), _ptr(table.device_index), table.size, raw.data_ptr(), n,
                                  U.data_ptr(), out.data_ptr(), st.data_ptr(), _lib.DAC_MODES[mode], ws, wsb, s)
        _lib.check(rc, "dr_sample_dac_from")
        if to_host:
            return finish_host(out, s)
        return out if device else out.cpu().numpy()
    k0, k1, off, offd = _stream_args(stream, n + 1)
    if kind == "ccf":
        rc = L.dr_sample_ccf(W.data_ptr(), _ptr(table.device_index), table.size, k0, k1, off, offd, n, U.data_ptr(), out.data_ptr(),
                             st.data_ptr(), ws, wsb, s)
    else:
        rc = L.dr_sample_dac(W.data_ptr(), _ptr(table.device_index), table.size, k0, k1, off, offd, n,
                             U.data_ptr(), out.data_ptr(), st.data_ptr(), _lib.DAC_MODES[mode], ws, wsb, s)
    _lib.check(rc, f"dr_sample_{kind}")
    if to_host:
        return finish_host(out, s)
    return out if device else out.cpu().numpy()


def ccf_sampler(table: WeightTable, n: int, stream, stats: OpStats | None = None,
                *, device: bool = False, out=None, uniforms_out=None):
    """Sorted uniforms + streaming merge: multinomial(w, n) in O(M + N) (samplers.py:255-259)."""
    return _sorted_sampler("ccf", table, n, stream, stats, device, out=out, U=uniforms_out)


def dac_sampler(table: WeightTable, n: int, stream, stats: OpStats | None = None,
                *, device: bool = False, mode: str = "auto", out=None, uniforms_out=None):
    """Sorted uniforms + divide-and-conquer (samplers.py:262-266).

    With a Philox stream this is one library call (``dr_sample_dac``): for
    N+1 <= 512 x (co-resident CTAs) a single cooperative kernel generates,
    scans and normalises the uniforms in registers and searches them.
    ``out`` / ``uniforms_out`` take preallocated CUDA buffers.
    """
    if mode not in _lib.DAC_MODES:
        raise ValueError(f"unknown mode {mode!r}")
    return _sorted_sampler("dac", table, n, stream, stats, device, mode, out=out, U=uniforms_out)


def warm_kernels() -> None:
    """Load the library and run every search kernel once (samplers.py:149-156)."""
    t = WeightTable([0.5, 1.0])
    u = torch.tensor([0.25, 0.75], dtype=torch.float64, device=_lib.device())
    ccf_match(u, t, check=False)
    dac_match(u, t, check=False)
    _lower_bounds(t, u)
    torch.cuda.current_stream().synchronize()
