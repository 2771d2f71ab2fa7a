"""ctypes boundary to libdrs.so (include/drs.h).

The library is loaded from this package directory (built in-tree by
``__graft_entry__.build()`` / ``make -C paper_2604_01356_b200/csrc``).  There is
no fallback: a missing library or a missing CUDA device raises immediately.
ctypes releases the GIL for the duration of every call; all calls are
stream-ordered on torch's current stream of the current device.
"""

from __future__ import annotations

import ctypes
import threading
from pathlib import Path

import torch

LIB_PATH = Path(__file__).resolve().with_name("libdrs.so")

# status bits (include/drs.h)
ST_INVALID_WEIGHT = 0x1
ST_DEGENERATE = 0x2
ST_ACCUM_OVERFLOW = 0x4
ST_NOT_SORTED = 0x8
ST_OUT_OF_SUPPORT = 0x10
ST_REPAIRED = 0x20
ST_NONFINITE = 0x40
ST_DECREASING = 0x80
ST_TOP_NOT_ONE = 0x100
ST_SHARD_CAPACITY = 0x200
ST_SHARD_WINDOW = 0x400

OP_TABLE = 1
OP_SORTED = 2

DAC_MODES = {"auto": 0, "merge": 1, "search": 2}

_c_void_p = ctypes.c_void_p
_i64 = ctypes.c_int64
_u64 = ctypes.c_uint64
_i32 = ctypes.c_int32
_int = ctypes.c_int
_size = ctypes.c_size_t
_dbl = ctypes.c_double

# name -> (restype, argtypes); mirrors include/drs.h
_PROTOS = {
    "dr_version": (ctypes.c_char_p, []),
    "dr_strerror": (ctypes.c_char_p, [_int]),
    "dr_device_accessible": (_int, [_c_void_p]),
    "dr_stream_synchronize": (_int, [_c_void_p]),
    "dr_scan_geometry": (None, [_c_void_p]),
    "dr_workspace_bytes": (_size, [_int, _i64, _i64, _i64]),
    "dr_workspace_init": (_int, [_c_void_p, _size, _c_void_p]),
    "dr_index_entries": (_i64, [_i64]),
    "dr_build_table": (_int, [_c_void_p, _i64, _c_void_p, _c_void_p, _c_void_p, _c_void_p, _size, _c_void_p]),
    "dr_build_table_log": (_int, [_c_void_p, _i64, _c_void_p, _c_void_p, _c_void_p, _c_void_p, _size, _c_void_p]),
    "dr_build_table_deferred": (_int, [_c_void_p, _i64, _c_void_p, _c_void_p, _c_void_p, _c_void_p, _size, _c_void_p]),
    "dr_build_table_log_deferred": (_int, [_c_void_p, _i64, _c_void_p, _c_void_p, _c_void_p, _c_void_p, _size,
                                           _c_void_p]),
    "dr_table_materialize": (_int, [_c_void_p, _c_void_p, _i64, _c_void_p, _c_void_p]),
    "dr_validate_table": (_int, [_c_void_p, _i64, _c_void_p, _c_void_p]),
    "dr_build_index": (_int, [_c_void_p, _i64, _c_void_p, _c_void_p]),
    "dr_uniforms": (_int, [_u64, _u64, _u64, _i64, _c_void_p, _c_void_p]),
    "dr_sorted_uniforms": (_int, [_u64, _u64, _u64, _i64, _c_void_p, _c_void_p, _c_void_p, _size, _c_void_p]),
    "dr_sorted_uniforms_from": (_int, [_c_void_p, _i64, _c_void_p, _c_void_p, _c_void_p, _size, _c_void_p]),
    "dr_match_binary": (_int, [_c_void_p, _c_void_p, _i64, _c_void_p, _i64, _c_void_p, _c_void_p]),
    "dr_sample_binary": (_int, [_c_void_p, _c_void_p, _i64, _u64, _u64, _u64, _i64, _c_void_p, _c_void_p]),
    "dr_sample_dac": (_int, [_c_void_p, _c_void_p, _i64, _u64, _u64, _u64, _c_void_p, _i64, _c_void_p, _c_void_p, _c_void_p, _i32, _c_void_p, _size, _c_void_p]),
    "dr_sample_dac_sync": (_int, [_c_void_p, _c_void_p, _i64, _u64, _u64, _u64, _c_void_p, _i64, _c_void_p, _c_void_p, _c_void_p, _i32, _c_void_p, _size, _c_void_p]),
    "dr_sample_dac_gather": (_int, [_c_void_p, _c_void_p, _i64, _u64, _u64, _u64, _c_void_p, _i64, _c_void_p, _c_void_p, _c_void_p, _i64, _i64, _i64, _c_void_p, _c_void_p, _i32, _c_void_p, _size, _c_void_p]),
    "dr_sample_dac_from": (_int, [_c_void_p, _c_void_p, _i64, _c_void_p, _i64, _c_void_p, _c_void_p, _c_void_p, _i32, _c_void_p, _size, _c_void_p]),
    "dr_sample_ccf": (_int, [_c_void_p, _c_void_p, _i64, _u64, _u64, _u64, _c_void_p, _i64, _c_void_p, _c_void_p, _c_void_p, _c_void_p, _size, _c_void_p]),
    "dr_sample_binary_dev": (_int, [_c_void_p, _c_void_p, _i64, _u64, _u64, _u64, _c_void_p, _i64, _c_void_p, _c_void_p]),
    "dr_match_ccf": (_int, [_c_void_p, _c_void_p, _i64, _c_void_p, _i64, _c_void_p, _c_void_p]),
    "dr_match_dac": (_int, [_c_void_p, _c_void_p, _i64, _c_void_p, _i64, _c_void_p, _i32, _c_void_p]),
    "dr_check_sorted_open": (_int, [_c_void_p, _i64, _c_void_p, _c_void_p]),
    "dr_lower_bound_range": (_int, [_c_void_p, _i64, _i64, _dbl, _c_void_p, _c_void_p]),
    "dr_resample_batched": (_int, [_c_void_p, _i64, _i64, _i64, _c_void_p, _i32, _c_void_p, _c_void_p, _c_void_p, _c_void_p, _c_void_p]),
    "dr_shard_scan": (_int, [_c_void_p, _i64, _c_void_p, _c_void_p, _c_void_p, _c_void_p, _size, _c_void_p]),
    "dr_shard_finalize": (_int, [_c_void_p, _i64, _c_void_p, _i32, _i32, _c_void_p, _c_void_p]),
    "dr_shard_scan_deferred": (_int, [_c_void_p, _i64, _c_void_p, _c_void_p, _c_void_p, _c_void_p, _c_void_p, _size,
                                      _c_void_p]),
    "dr_shard_finalize_deferred": (_int, [_i64, _c_void_p, _i32, _i32, _c_void_p, _c_void_p]),
    "dr_shard_range": (_int, [_c_void_p, _i64, _c_void_p, _i32, _i32, _c_void_p, _c_void_p]),
    "dr_shard_unif_totals": (_int, [_u64, _u64, _u64, _i64, _i64, _i64, _c_void_p, _c_void_p, _c_void_p]),
    "dr_shard_unif_local": (_int, [_u64, _u64, _u64, _i64, _c_void_p, _c_void_p, _i64, _c_void_p, _i32, _i32,
                                   _c_void_p, _i64, _i64, _i32, _c_void_p, _c_void_p, _c_void_p, _size,
                                   _c_void_p]),
    "dr_gather_rows": (_int, [_c_void_p, _i64, _i64, _c_void_p, _i64, _i64, _c_void_p, _c_void_p, _c_void_p]),
    "dr_histogram": (_int, [_c_void_p, _i64, _i64, _c_void_p, _c_void_p, _c_void_p]),
    "dr_chi_square_workspace": (_size, [_i64]),
    "dr_chi_square": (_int, [_c_void_p, _c_void_p, _i64, _i64, _c_void_p, _c_void_p, _size, _c_void_p]),
    "dr_op_counts": (_int, [_i32, _c_void_p, _i64, _c_void_p, _i64, _c_void_p, _c_void_p, _c_void_p]),
    "dr_shard_match": (_int, [_c_void_p, _c_void_p, _i64, _i64, _c_void_p, _i64, _c_void_p, _c_void_p, _c_void_p]),
}

_lib = None
_lib_lock = threading.Lock()


def load_library(path: Path | str | None = None):
    """Load libdrs.so and bind the prototypes; raises if it is missing."""
    global _lib
    with _lib_lock:
        if _lib is not None and path is None:
            return _lib
        p = Path(path) if path is not None else LIB_PATH
        if not p.exists():
            raise RuntimeError(
                f"{p} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
                "(there is no CPU fallback)"
            )
        lib = ctypes.CDLL(str(p))
        for name, (res, args) in _PROTOS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if path is None:
            _lib = lib
        return lib


_cuda_ok = False


def lib():
    """The bound library, after checking (once) that a CUDA device is present."""
    global _cuda_ok
    if not _cuda_ok:
        if not torch.cuda.is_available():
            raise RuntimeError("paper_2604_01356_b200 needs a CUDA device (sm_100a); none is visible")
        _cuda_ok = True
    return _lib if _lib is not None else load_library()


def check(rc: int, what: str) -> None:
    if rc != 0:
        msg = load_library().dr_strerror(rc).decode()
        raise RuntimeError(f"{what} failed: {msg} ({rc})")


_accessible: dict[int, bool] = {}


def device_accessible(ptr: int) -> bool:
    """True when the device can dereference ``ptr`` itself (pinned host memory under UVA)."""
    ok = _accessible.get(ptr)
    if ok is None:
        ok = bool(lib().dr_device_accessible(ptr))
        _accessible[ptr] = ok
    return ok


_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None)


def stream_handle() -> int:
    """cudaStream_t of torch's current stream on the current device."""
    if _raw_stream is not None:
        return _raw_stream(torch.cuda.current_device())
    return torch.cuda.current_stream().cuda_stream


def device() -> torch.device:
    return torch.device("cuda", torch.cuda.current_device())


def scan_geometry() -> tuple[int, ...]:
    g = (ctypes.c_int32 * 6)()
    load_library().dr_scan_geometry(ctypes.cast(g, ctypes.c_void_p))
    return tuple(int(v) for v in g)


class _Workspace:
    __slots__ = ("tensor", "nbytes")

    def __init__(self):
        self.tensor = None
        self.nbytes = 0


_ws: dict[tuple[int, int], _Workspace] = {}
_ws_lock = threading.Lock()
# superseded workspaces stay allocated: a CUDA graph captured earlier on the
# stream may still point at them
_ws_retired: list = []


_ws_bytes: dict[tuple[int, int], int] = {}


def workspace_bytes(op: int, n: int) -> int:
    """dr_workspace_bytes(op, n, n, 0), memoised (a pure function of its arguments)."""
    v = _ws_bytes.get((op, n))
    if v is None:
        v = int(lib().dr_workspace_bytes(op, n, n, 0))
        _ws_bytes[(op, n)] = v
    return v


def workspace(nbytes: int, st: int | None = None) -> tuple[int, int]:
    """(pointer, size) of the scan workspace of the current (device, stream).

    Grown on demand; a new allocation is initialised with dr_workspace_init
    on the stream it will be used on.
    """
    dev = torch.cuda.current_device()
    if st is None:
        st = stream_handle()
    with _ws_lock:
        w = _ws.setdefault((dev, st), _Workspace())
        if w.nbytes < nbytes:
            size = max(nbytes, 2 * w.nbytes, 1 << 16)
            if w.tensor is not None:
                _ws_retired.append(w.tensor)
            w.tensor = torch.empty(size, dtype=torch.uint8, device=device())
            w.nbytes = size
            check(lib().dr_workspace_init(w.tensor.data_ptr(), size, st), "dr_workspace_init")
        return w.tensor.data_ptr(), w.nbytes
