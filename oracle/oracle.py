"""numpy wrappers over libdrs_oracle.so -- TEST INFRASTRUCTURE ONLY.

Importable only from tests/, __graft_entry__.smoke() and bench.py's CPU
baseline legs.  Never used by the product package.
"""

from __future__ import annotations

import ctypes
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "libdrs_oracle.so"

_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_U64 = ctypes.c_uint64
_INT = ctypes.c_int
_D = ctypes.c_double

_PROTOS = {
    "drs_ref_raw_draw": (_U64, [_U64, _U64, _U64]),
    "drs_ref_u01": (_D, [_U64]),
    "drs_ref_uniforms": (None, [_U64, _U64, _U64, _I64, _P]),
    "drs_ref_log": (_D, [_D]),
    "drs_ref_neglog_array": (None, [_P, _I64, _P]),
    "drs_ref_chain_scan": (None, [_P, _I64, _INT, _P, _P]),
    "drs_ref_build_table": (_INT, [_P, _I64, _P]),
    "drs_ref_exp": (_D, [_D]),
    "drs_ref_exp_array": (None, [_P, _I64, _P]),
    "drs_ref_build_table_log": (_INT, [_P, _I64, _P]),
    "drs_ref_sorted_from_z": (_INT, [_P, _I64, _P]),
    "drs_ref_sorted_uniforms": (_INT, [_U64, _U64, _U64, _I64, _P]),
    "drs_ref_sorted_uniforms_from": (_INT, [_P, _I64, _P]),
    "drs_ref_index_entries": (_I64, [_I64]),
    "drs_ref_search_entries": (_I64, [_I64]),
    "drs_ref_build_table_deferred": (_INT, [_P, _I64, _P, _P, _P]),
    "drs_ref_index_l1_local": (_INT, [_P, _I64, _P]),
    "drs_ref_build_index": (None, [_P, _I64, _P]),
    "drs_ref_build_table_sharded": (_INT, [_P, _I64, _INT, _P, _P]),
    "drs_ref_resample_batched": (_INT, [_P, _I64, _I64, _I64, _P, _P, _P, _P]),
    "drs_port_total": (_D, [_P, _I64]),
    "drs_port_build_table": (_INT, [_P, _I64, _P]),
    "drs_port_upper_bound": (_I64, [_P, _I64, _I64, _D]),
    "drs_port_match_binary": (None, [_P, _I64, _P, _I64, _P]),
    "drs_port_match_ccf": (None, [_P, _I64, _P, _I64, _P]),
    "drs_port_match_dac": (_INT, [_P, _I64, _P, _I64, _P]),
    "drs_port_repair_open_strict": (None, [_P, _I64]),
    "drs_port_sorted_from_z": (_INT, [_P, _I64, _P]),
    "drs_port_sorted_uniforms": (_INT, [_U64, _U64, _U64, _I64, _P]),
    "drs_port_sampler": (_INT, [_INT, _P, _I64, _U64, _U64, _U64, _I64, _P, _P]),
    "drs_port_throughput": (_D, [_INT, _P, _I64, _I64, _INT, _INT, _U64, _U64]),
    "drs_port_batched_throughput": (_D, [_P, _I64, _I64, _I64, _INT, _INT, _U64, _U64]),
}

_lib = None


def build() -> Path:
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB


def lib():
    global _lib
    if _lib is None:
        if not LIB.exists():
            build()
        L = ctypes.CDLL(str(LIB))
        for name, (res, args) in _PROTOS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


SAMPLER_IDS = {"dac": 0, "ccf": 1, "binary": 2}


def key_of(seed, spawn_key=()):
    k = np.random.SeedSequence(int(seed), spawn_key=tuple(spawn_key)).generate_state(2, np.uint64)
    return int(k[0]), int(k[1])


def uniforms(k0, k1, offset, k):
    out = np.empty(int(k), dtype=np.float64)
    lib().drs_ref_uniforms(k0, k1, offset, int(k), _p(out))
    return out


def log(x):
    x = _f64(x)
    out = np.empty_like(x)
    for i, v in enumerate(x.ravel()):
        out.ravel()[i] = lib().drs_ref_log(float(v))
    return out


def neglog(u):
    u = _f64(u)
    z = np.empty_like(u)
    lib().drs_ref_neglog_array(_p(u), u.size, _p(z))
    return z


def chain_scan(x, K):
    x = _f64(x)
    S = np.empty_like(x)
    tot = np.zeros(1)
    lib().drs_ref_chain_scan(_p(x), x.size, int(K), _p(S), _p(tot))
    return S, float(tot[0])


def build_table(w):
    w = _f64(w)
    W = np.empty_like(w)
    st = lib().drs_ref_build_table(_p(w), w.size, _p(W))
    return W, int(st)


def port_build_table(w):
    w = _f64(w)
    W = np.empty_like(w)
    st = lib().drs_port_build_table(_p(w), w.size, _p(W))
    return W, int(st)


def port_total(w):
    w = _f64(w)
    return float(lib().drs_port_total(_p(w), w.size))


def build_table_sharded(w, G):
    w = _f64(w)
    W = np.empty_like(w)
    T = np.empty(int(G))
    st = lib().drs_ref_build_table_sharded(_p(w), w.size, int(G), _p(W), _p(T))
    return W, T, int(st)


def sorted_uniforms(k0, k1, offset, n):
    U = np.empty(int(n), dtype=np.float64)
    st = lib().drs_ref_sorted_uniforms(k0, k1, offset, int(n), _p(U))
    return U, int(st)


def sorted_uniforms_from(raw, n):
    raw = _f64(raw)
    U = np.empty(int(n), dtype=np.float64)
    st = lib().drs_ref_sorted_uniforms_from(_p(raw), int(n), _p(U))
    return U, int(st)


def sorted_from_z(z, n, association="device"):
    z = _f64(z).copy()
    U = np.empty(int(n), dtype=np.float64)
    fn = lib().drs_ref_sorted_from_z if association == "device" else lib().drs_port_sorted_from_z
    st = fn(_p(z), int(n), _p(U))
    return U, int(st)


def port_sorted_uniforms(k0, k1, offset, n):
    U = np.empty(int(n), dtype=np.float64)
    st = lib().drs_port_sorted_uniforms(k0, k1, offset, int(n), _p(U))
    return U, int(st)


def build_index(W):
    W = _f64(W)
    out = np.empty(int(lib().drs_ref_index_entries(W.size)), dtype=np.float64)
    lib().drs_ref_build_index(_p(W), W.size, _p(out))
    return out


def search_entries(M):
    """doubles of the index the searches descend (levels + top guide)"""
    return int(lib().drs_ref_search_entries(int(M)))


def build_table_deferred(w):
    """dr_build_table_deferred's outputs: (V in-tile sums, full idx with the
    header and tile pairs, W, status)."""
    w = _f64(w)
    V = np.empty(w.size, dtype=np.float64)
    W = np.empty(w.size, dtype=np.float64)
    idx = np.empty(int(lib().drs_ref_index_entries(w.size)), dtype=np.float64)
    st = lib().drs_ref_build_table_deferred(_p(w), w.size, _p(V), _p(idx), _p(W))
    return V, idx, W, int(st)


def index_l1_local(V, idx):
    """The index of a deferred table whose level 1 keeps in-tile values (top
    guide above level 1): idx (a copy) with level 1 = V at the block ends;
    (idx, True) when that applies, else (idx, False)."""
    V = _f64(V)
    idx = np.array(idx, dtype=np.float64, copy=True)
    done = lib().drs_ref_index_l1_local(_p(V), V.size, _p(idx))
    return idx, bool(done)


def match(kind, W, u):
    W = _f64(W)
    u = _f64(u)
    out = np.empty(u.size, dtype=np.int64)
    if u.size == 0:
        return out
    if kind == "binary":
        lib().drs_port_match_binary(_p(W), W.size, _p(u), u.size, _p(out))
    elif kind == "ccf":
        lib().drs_port_match_ccf(_p(W), W.size, _p(u), u.size, _p(out))
    else:
        rc = lib().drs_port_match_dac(_p(W), W.size, _p(u), u.size, _p(out))
        if rc:
            raise RuntimeError("dac stack overflow")
    return out


def upper_bound(W, lo, hi, x):
    W = _f64(W)
    return int(lib().drs_port_upper_bound(_p(W), int(lo), int(hi), float(x)))


def repair_open_strict(u):
    u = _f64(u).copy()
    lib().drs_port_repair_open_strict(_p(u), u.size)
    return u


def resample_batched(w, n, keys):
    w = _f64(w)
    B, Mf = w.shape
    keys = np.ascontiguousarray(keys, dtype=np.uint64).reshape(B, 3)
    W = np.empty_like(w)
    U = np.empty((B, int(n)), dtype=np.float64)
    out = np.empty((B, int(n)), dtype=np.int64)
    st = lib().drs_ref_resample_batched(_p(w), B, Mf, int(n), _p(keys), _p(W), _p(U), _p(out))
    return out, U, W, int(st)


def port_sampler(which, W, k0, k1, offset, N):
    W = _f64(W)
    scratch = np.empty(2 * int(N) + 2, dtype=np.float64)
    out = np.empty(int(N), dtype=np.int64)
    lib().drs_port_sampler(SAMPLER_IDS[which], _p(W), W.size, k0, k1, offset, int(N), _p(scratch), _p(out))
    return out


def port_throughput(which, W, N, threads, calls, k0, k1):
    W = _f64(W)
    return float(lib().drs_port_throughput(SAMPLER_IDS[which], _p(W), W.size, int(N), int(threads), int(calls), k0, k1))


def port_batched_throughput(w, Nf, threads, reps, k0, k1):
    """Wall seconds of the reference's per-filter loop over the rows of w."""
    w = _f64(w)
    B, Mf = w.shape
    return float(lib().drs_port_batched_throughput(_p(w), B, Mf, int(Nf), int(threads), int(reps), k0, k1))


def exp(x):
    x = _f64(x)
    y = np.empty_like(x)
    lib().drs_ref_exp_array(_p(x), x.size, _p(y))
    return y


def build_table_log(lw):
    lw = _f64(lw)
    W = np.empty_like(lw)
    st = lib().drs_ref_build_table_log(_p(lw), lw.size, _p(W))
    return W, int(st)
