"""GPU parity: the CUDA path through the C ABI against the oracle and the reference.

Exact mode: given the reference's own W and U, every sampler's indices must
equal the reference's bit for bit.  Device mode: W and U computed on the GPU
must equal the oracle's device-association twins bit for bit, and differ
from the reference only by fp64 reassociation (ulp drift reported; index
flips only where u sits within the drift of a boundary).
"""

import numpy as np
import pytest
import torch

from tests.helpers import (
    PhiloxStream,
    ReplayStream,
    boundary_query_set,
    enumerate_weight_tables,
    golden_cases,
    linear_scan_bulk,
    reference_table_exact,
    ulps,
)

pytestmark = pytest.mark.gpu


def dev(a):
    return torch.as_tensor(np.asarray(a, dtype=np.float64), device="cuda")


# ---------------------------------------------------------------- exact mode
def test_exact_mode_reference_cases(drs, golden):
    n = 0
    for W, u, e in golden_cases(golden):
        t = drs.WeightTable(W)
        np.testing.assert_array_equal(drs.ccf_match(u, t), e)
        np.testing.assert_array_equal(drs.dac_match(u, t), e)
        np.testing.assert_array_equal(drs.dac_match(u, t, mode="merge"), e)
        np.testing.assert_array_equal(drs.dac_match(u, t, mode="search"), e)
        np.testing.assert_array_equal(drs.binary_sampler(t, u.shape[0], ReplayStream(u)), e)
        n += 1
    assert n == 300


def test_exact_mode_exhaustive_tables(drs):
    for raw in enumerate_weight_tables(6):
        W = reference_table_exact(raw)
        t = drs.WeightTable(W)
        u = boundary_query_set(W)
        e = linear_scan_bulk(W, u)
        np.testing.assert_array_equal(drs.ccf_match(u, t), e)
        np.testing.assert_array_equal(drs.dac_match(u, t, mode="merge"), e)
        np.testing.assert_array_equal(drs.dac_match(u, t, mode="search"), e)
        np.testing.assert_array_equal(drs.binary_sampler(t, u.shape[0], ReplayStream(u)), e)


def test_exact_mode_c1(drs, golden, orc):
    W = golden[f"tbl_cum_{int(golden['tbl_count']) - 1}"]
    t = drs.WeightTable(W)
    d = PhiloxStream(2001).uniforms(1025)
    U, _ = orc.sorted_from_z(-np.log(d), 1024, association="port")  # the reference's U
    np.testing.assert_array_equal(drs.dac_match(U, t), golden["c1_dac"])
    np.testing.assert_array_equal(drs.ccf_match(U, t), golden["c1_ccf"])
    np.testing.assert_array_equal(drs.binary_sampler(t, 1024, ReplayStream(d[:1024])), golden["c1_binary"])


def test_exact_mode_large_random(drs, orc):
    rng = np.random.default_rng(77)
    for M, N in [(1 << 20, 1 << 20), (1 << 22, 1 << 14), (300001, 4097), (5, 100000)]:
        w = np.exp(3 * rng.standard_normal(M))
        w[rng.random(M) < 0.2] = 0.0
        W, _ = orc.port_build_table(w)
        U = np.sort(rng.random(N))
        U = U[U > 0]
        k = min(N // 4, M)
        U[: k] = np.sort(rng.choice(W[W > 0], size=k))  # exact boundaries
        U = np.sort(U)
        e = orc.match("binary", W, U)
        t = drs.WeightTable(W)
        Ud = dev(U)
        for mode in ("merge", "search", "auto"):
            np.testing.assert_array_equal(drs.dac_match(Ud, t, check=False, mode=mode).cpu().numpy(), e)
        np.testing.assert_array_equal(drs.ccf_match(Ud, t, check=False).cpu().numpy(), e)
        perm = rng.permutation(U.shape[0])
        np.testing.assert_array_equal(drs.binary_sampler(t, U.shape[0], ReplayStream(U[perm])), e[perm])


@pytest.mark.parametrize("M,N,frac,blk", [
    ((1 << 22) + 3, 600_000, 0.5, 3000),   # M >> N: tiles without a u chunk (bisection), split runs
    ((1 << 20) + 7, 1 << 20, 0.6, 5000),   # M ~ N: merge path, split runs
    (1 << 20, 70_001, 0.97, 1),            # one weight holds 97% of the mass: one run spans the u's
    ((1 << 18) + 1, 300_000, 0.3, 20000),  # a heavy block spanning several tiles
])
@pytest.mark.parametrize("paths_min", [None, "64"])
def test_merge_heavy_runs(drs, orc, M, N, frac, blk, paths_min, monkeypatch):
    """Tiles whose u-run is longer than MT_HEAVY: the tile CTA handles the
    ragged ends, k_merge_heavy the whole chunks inside; bit-exact against the
    oracle's lower bounds with exact boundaries inside the heavy block, for
    CCF and DaC in merge mode, with ragged N.  Both tile bodies: the per-u
    bisection of the staged tile (the default: measured never slower) and the
    linear merge path from 64 u's per tile (DRS_MERGE_PATHS_MIN=64)."""
    if paths_min:
        monkeypatch.setenv("DRS_MERGE_PATHS_MIN", paths_min)
    else:
        monkeypatch.delenv("DRS_MERGE_PATHS_MIN", raising=False)
    rng = np.random.default_rng(79)
    w = np.exp(rng.standard_normal(M))
    off = int(rng.integers(0, M - blk))
    w[off:off + blk] = (w.sum() - w[off:off + blk].sum()) * frac / (1 - frac) / blk
    W, _ = orc.port_build_table(w)
    U = rng.random(N)
    U[: N // 8] = rng.choice(W[off:off + blk], size=N // 8)  # exact boundaries in the heavy block
    U = np.sort(U[U > 0])
    e = orc.match("binary", W, U)
    t = drs.WeightTable(W)
    Ud = dev(U)
    np.testing.assert_array_equal(drs.ccf_match(Ud, t, check=False).cpu().numpy(), e)
    np.testing.assert_array_equal(drs.dac_match(Ud, t, check=False, mode="merge").cpu().numpy(), e)
    # host input and result (U has ties, so the strict sortedness check is off)
    np.testing.assert_array_equal(drs.ccf_match(U, t, check=False), e)


def test_exact_mode_many_u_throughput_search(drs, orc):
    """Millions of u's: the index search switches to its throughput variant
    (four u's per thread, half-node reads); bit-exact against the oracle's
    lower bounds, with exact boundaries, ties, zero runs, u = 1 and the clamp."""
    rng = np.random.default_rng(78)
    M, N = (1 << 22) + 5, 3_000_000
    w = np.exp(2 * rng.standard_normal(M))
    w[rng.random(M) < 0.3] = 0.0
    w[-3:] = 0.0  # trailing zeros: u = 1 maps to the first index of the top run
    W, _ = orc.port_build_table(w)
    U = rng.random(N)
    U[: N // 4] = rng.choice(W[W > 0], size=N // 4)  # exact boundaries
    U[:1000] = 1.0
    U = np.sort(U[U > 0])
    e = orc.match("binary", W, U)
    t = drs.WeightTable(W)
    Ud = dev(U)
    np.testing.assert_array_equal(drs.dac_match(Ud, t, check=False, mode="search").cpu().numpy(), e)
    np.testing.assert_array_equal(drs.samplers._lower_bounds(t, Ud).cpu().numpy(), e)
    # unsorted u (the binary matcher's input order)
    perm = rng.permutation(U.shape[0])
    np.testing.assert_array_equal(drs.samplers._lower_bounds(t, dev(U[perm])).cpu().numpy(), e[perm])


def test_clamp_and_ties(drs):
    t = drs.WeightTable([0.25, 0.25, 0.5, 1.0, 1.0, 1.0])
    u = np.array([1e-300, 0.25, 0.2500000001, 0.5, 1.0])
    e = np.array([0, 0, 2, 2, 3])
    np.testing.assert_array_equal(drs.ccf_match(u, t), e)
    np.testing.assert_array_equal(drs.dac_match(u, t, mode="search"), e)
    # u > 1 (check=False): the reference's bisection clamps to M-1
    ud = dev([0.9, 1.5])
    assert drs.dac_match(ud, t, check=False, mode="search").tolist() == [3, 5]
    assert drs.dac_match(ud, t, check=False, mode="merge").tolist() == [3, 5]


# --------------------------------------------------------------- device mode
def test_build_table_bit_exact_vs_oracle(drs, orc, golden):
    for i in range(int(golden["tbl_count"])):
        raw = golden[f"tbl_raw_{i}"]
        t = drs.build_weight_table(raw)
        W, _ = orc.build_table(raw)
        np.testing.assert_array_equal(t.cum, W)
        # the single-pass (deferred) table: values, index, header and tile pairs
        np.testing.assert_array_equal(t.device_index.cpu().numpy(), orc.build_table_deferred(raw)[1])
        t2 = drs.build_weight_table(raw, deferred=False)  # the two-pass table
        np.testing.assert_array_equal(t2.cum, W)
        np.testing.assert_array_equal(t2.device_index.cpu().numpy(), orc.build_index(W))
        ref = golden[f"tbl_cum_{i}"]
        assert np.abs(t.cum - ref).max() <= 1e-12


@pytest.mark.parametrize("M", [1, 2, 31, 33, 8447, 8448, 8449, 3 * 8448 + 5, 1 << 20, (1 << 22) + 3])
def test_build_table_tile_edges(drs, orc, M):
    rng = np.random.default_rng(M)
    w = rng.random(M)
    w[rng.random(M) < 0.1] = 0.0
    if w.sum() == 0:
        w[0] = 1
    t = drs.build_weight_table(w)
    W, _ = orc.build_table(w)
    np.testing.assert_array_equal(t.cum, W)
    assert t.cum[-1] == 1.0 and np.all(np.diff(t.cum) >= 0)


def test_build_table_errors(drs):
    with pytest.raises(ValueError, match="empty distribution"):
        drs.build_weight_table([])
    with pytest.raises(ValueError, match="empty distribution"):
        drs.build_weight_table(np.ones((2, 2)))
    with pytest.raises(ValueError, match="degenerate distribution"):
        drs.build_weight_table([0.0, 0.0])
    for bad in ([-1.0, 2.0], [np.nan], [np.inf, 1.0]):
        with pytest.raises(ValueError, match="invalid weight"):
            drs.build_weight_table(bad)
    with pytest.raises(ValueError, match="accumulation overflow"):
        drs.build_weight_table([1e308, 1e308])


def test_sorted_uniforms_bit_exact_vs_oracle(drs, orc, golden):
    for i, (seed, n) in enumerate(golden["su_cases"]):
        s = drs.RngStream(int(seed))
        U = drs.sorted_uniforms(s, int(n))
        assert s.draws == int(n) + 1
        k0, k1 = orc.key_of(int(seed))
        Uo, _ = orc.sorted_uniforms(k0, k1, 0, int(n))
        np.testing.assert_array_equal(U, Uo)
        # against the reference (PCG64 replaced by the same Philox draws): reassociation + log ulp only
        ref = golden[f"su_U_{i}"]
        assert np.abs(U - ref).max() <= 1e-13


@pytest.mark.parametrize("n", [1, 2, 3, 1022, 1023, 1024, 1025, 4095, 70001, 75775, 75776, 150000, 227327, 227328, 303104, 1 << 20])
def test_sorted_uniforms_sizes(drs, orc, n):
    s = drs.RngStream(n, (3,))
    s.uniforms(5)  # non-multiple-of-4 draw offset
    U = drs.sorted_uniforms(s, n)
    k0, k1 = orc.key_of(n, (3,))
    Uo, _ = orc.sorted_uniforms(k0, k1, 5, n)
    np.testing.assert_array_equal(U, Uo)
    assert U[0] > 0 and U[-1] < 1 and np.all(np.diff(U) > 0)


@pytest.mark.parametrize("n", [1, 2, 1023, 1025, 4095, 70001, 150000, 227327])
def test_sorted_uniforms_pipeline_small_n(drs, orc, golden, n, monkeypatch):
    """n + 1 spacings that fit a co-resident grid (up to three 512-spacing tiles per SM: 227,328 on a
    148-SM part) take ONE cooperative launch (k_dac_fused<false>: no table);
    DRS_NO_FUSED_UNIFORMS=1 selects the pass 1 /
    chain / pass 2 / finalize pipeline that larger n always use: same U, same
    repair, same stream advance."""
    k0, k1 = orc.key_of(n, (3,))
    Uo, _ = orc.sorted_uniforms(k0, k1, 5, n)
    for env in (None, "1"):
        if env:
            monkeypatch.setenv("DRS_NO_FUSED_UNIFORMS", env)
        else:
            monkeypatch.delenv("DRS_NO_FUSED_UNIFORMS", raising=False)
        s = drs.RngStream(n, (3,))
        s.uniforms(5)
        np.testing.assert_array_equal(drs.sorted_uniforms(s, n), Uo)
        assert s.draws == 5 + n + 1
    monkeypatch.setenv("DRS_NO_FUSED_UNIFORMS", "1")
    for i in range(int(golden["rp_count"])):  # the replayed collapse / repair cases through the pipeline
        d = golden[f"rp_draws_{i}"]
        U = drs.sorted_uniforms(ReplayStream(d), d.shape[0] - 1)
        np.testing.assert_array_equal(U, orc.sorted_uniforms_from(d, d.shape[0] - 1)[0])


def test_replay_and_repair_bit_exact(drs, orc, golden):
    for i in range(int(golden["rp_count"])):
        d = golden[f"rp_draws_{i}"]
        n = d.shape[0] - 1
        U = drs.sorted_uniforms(ReplayStream(d), n)
        Uo, _ = orc.sorted_uniforms_from(d, n)
        np.testing.assert_array_equal(U, Uo)
        assert U[0] > 0 and U[-1] < 1 and np.all(np.diff(U) > 0)
        assert np.abs(U - golden[f"rp_U_{i}"]).max() <= 1e-12
    u = drs.sorted_uniforms(ReplayStream([0.5, 0.5, 0.5]), 2)
    np.testing.assert_allclose(u, [1 / 3, 2 / 3], rtol=1e-15)


def test_repair_many_sites(drs, orc):
    rng = np.random.default_rng(5)
    d = rng.random(50001)
    d[rng.random(50001) < 0.3] = 1 - 2.0 ** -53  # thousands of vanishing spacings
    U = drs.sorted_uniforms(ReplayStream(d), 50000)
    Uo, st = orc.sorted_uniforms_from(d, 50000)
    assert st & 0x20
    np.testing.assert_array_equal(U, Uo)


def test_uniforms_match_numpy_philox(drs):
    s = drs.RngStream(2003)
    a = s.uniforms(7)
    b = s.uniforms(1000)
    gen = np.random.Generator(np.random.Philox(np.random.SeedSequence(2003)))
    np.testing.assert_array_equal(np.concatenate([a, b]), gen.random(1007))
    assert s.draws == 1007


def test_binary_sampler_bit_exact_vs_oracle(drs, orc):
    w = np.exp(2 * np.random.default_rng(8).standard_normal(100000))
    t = drs.build_weight_table(w)
    s = drs.RngStream(31)
    s.uniforms(3)
    out = drs.binary_sampler(t, 50001, s)
    k0, k1 = orc.key_of(31)
    u = orc.uniforms(k0, k1, 3, 50001)
    np.testing.assert_array_equal(out, orc.match("binary", t.cum, u))


@pytest.mark.parametrize("M,N", [(65536, 1024), (1 << 20, 1 << 20), (1 << 24, 1 << 12), (1000, 1 << 18)])
def test_samplers_device_mode_vs_oracle(drs, orc, M, N):
    w = np.exp(np.random.default_rng(M + N).standard_normal(M))
    t = drs.build_weight_table(w)
    W, _ = orc.build_table(w)
    np.testing.assert_array_equal(t.cum, W)
    k0, k1 = orc.key_of(N)
    Uo, _ = orc.sorted_uniforms(k0, k1, 0, N)
    e = orc.match("dac", W, Uo)
    for fn in (drs.dac_sampler, drs.ccf_sampler):
        np.testing.assert_array_equal(fn(t, N, drs.RngStream(N)), e)
    for mode in ("merge", "search"):
        np.testing.assert_array_equal(drs.dac_sampler(t, N, drs.RngStream(N), mode=mode), e)


def test_device_vs_reference_flips_only_near_boundaries(drs, orc):
    """Device-mode disagreement with the reference association is confined to
    u within the measured reassociation drift of a boundary W_j."""
    M, N = 1 << 20, 1 << 16
    w = np.exp(4 * np.random.default_rng(1003).standard_normal(M))
    t = drs.build_weight_table(w)
    Wref, _ = orc.port_build_table(w)
    s = drs.RngStream(2003)
    U = drs.sorted_uniforms(drs.RngStream(2003), N)
    d = PhiloxStream(2003).uniforms(N + 1)
    Uref, _ = orc.sorted_from_z(-np.log(d), N, association="port")
    out = drs.dac_sampler(t, N, s)
    eref = orc.match("dac", Wref, Uref)
    drift_W = np.abs(t.cum - Wref).max()
    drift_U = np.abs(U - Uref).max()
    flips = np.nonzero(out != eref)[0]
    near = np.abs(Wref[eref[flips]] - Uref[flips]) <= 2 * (drift_W + drift_U) + 1e-300
    near |= np.abs(Wref[np.maximum(eref[flips] - 1, 0)] - Uref[flips]) <= 2 * (drift_W + drift_U)
    assert near.all(), (flips, drift_W, drift_U)


def test_chi_square_counts(drs):
    rng = np.random.default_rng(40)
    for raw in (rng.random(16), np.full(16, 1 / 16)):
        t = drs.build_weight_table(raw)
        expected = 1_000_000 * t.weights()
        for fn in (drs.binary_sampler, drs.ccf_sampler, drs.dac_sampler):
            counts = np.bincount(fn(t, 1_000_000, drs.RngStream(41)), minlength=16)
            chi2 = float(((counts - expected) ** 2 / expected).sum())
            assert chi2 < 37.70


def test_zero_weight_never_drawn(drs):
    t = drs.build_weight_table([0.0, 0.3, 0.0, 0.7, 0.0])
    for fn in (drs.binary_sampler, drs.ccf_sampler, drs.dac_sampler):
        c = np.bincount(fn(t, 1_000_000, drs.RngStream(17)), minlength=5)
        assert c[[0, 2, 4]].sum() == 0


# ---------------------------------------------------------- batched / sharded
def test_batched_bit_exact_vs_oracle(drs, orc):
    rng = np.random.default_rng(1004)
    B, Mf, Nf = 64, 16384, 256
    pi = rng.dirichlet(np.ones(64), size=B)
    q = rng.chisquare(6, size=(B, 256, 64))
    w = np.exp(np.log(1 / 256) + np.log(pi)[:, None, :] - 0.5 * q).reshape(B, Mf)
    streams = [drs.RngStream(2004, (b,)) for b in range(B)]
    for s in streams[::3]:
        s.uniforms(1)
    keys = np.array([[s.key[0], s.key[1], s.position] for s in streams], dtype=np.uint64)
    out, U, W = drs.resample_batched(w, Nf, streams, return_uniforms=True, return_tables=True)
    eo, Uo, Wo, st = orc.resample_batched(w, Nf, keys)
    np.testing.assert_array_equal(W, Wo)
    np.testing.assert_array_equal(U, Uo)
    np.testing.assert_array_equal(out, eo)
    # identical to the single-filter path
    t = drs.build_weight_table(w[5])
    np.testing.assert_array_equal(t.cum, W[5])


@pytest.mark.parametrize("B,Mf,Nf", [(300, 16384, 256), (333, 16383, 257), (7, 12000, 3000), (5, 1, 4),
                                     (200, 33, 1), (4, 8449, 1023), (3, 25000, 0),
                                     # row and tile edges, one and two tiles, many filters per SM
                                     (157, 16896, 511), (150, 2, 1), (149, 34, 5), (200, 1056, 64),
                                     (200, 1058, 63), (211, 8448, 100), (211, 8450, 300), (90, 9504, 200),
                                     (50, 4096, 0), (400, 16000, 130), (160, 8448, 330), (160, 8448, 400)])
def test_batched_shapes_vs_oracle(drs, orc, B, Mf, Nf):
    """Tile edges, odd M_f (no TMA path), several table / uniform tiles, more
    filters than resident CTAs, N_f = 0; bit-exact against the oracle."""
    rng = np.random.default_rng(B * 7 + Mf)
    w = np.exp(2.0 * rng.standard_normal((B, Mf)))
    w[rng.random((B, Mf)) < 0.1] = 0.0
    w[:, -1] += 1.0  # no degenerate filter
    streams = [drs.RngStream(99, (b,)) for b in range(B)]
    keys = np.array([[s.key[0], s.key[1], s.position] for s in streams], dtype=np.uint64)
    res = drs.resample_batched(w, Nf, streams, return_uniforms=True, return_tables=True)
    eo, Uo, Wo, st = orc.resample_batched(w, Nf, keys)
    np.testing.assert_array_equal(res[2], Wo)
    np.testing.assert_array_equal(res[1], Uo)
    np.testing.assert_array_equal(res[0], eo)
    assert all(s.position == (Nf + 1 if Nf else 0) for s in streams)


@pytest.mark.parametrize("case", ["heavy_chunk", "zero_rows", "spike_first", "no_tables"])
def test_batched_mass_layouts(drs, orc, case):
    """Many draws in one chunk, whole zero rows, mass in the first or last
    entry, and the index-only call (no W / U outputs), over more filters than
    resident CTAs."""
    rng = np.random.default_rng(["heavy_chunk", "zero_rows", "spike_first", "no_tables"].index(case))
    B, Mf, Nf = 700, 16384, 256
    w = np.exp(rng.standard_normal((B, Mf)))
    if case == "heavy_chunk":
        w[:, 5000] = 1e6
        w[::2, 16383] = 1e6
    elif case == "zero_rows":
        w[:, 1056:3168] = 0.0
        w[:, :40] = 0.0
        w[:, 16000:] = 0.0
    elif case == "spike_first":
        w[:, 0] = 1e9
    streams = [drs.RngStream(7, (b,)) for b in range(B)]
    keys = np.array([[s.key[0], s.key[1], s.position] for s in streams], dtype=np.uint64)
    eo, Uo, Wo, st = orc.resample_batched(w, Nf, keys)
    if case == "no_tables":
        out = drs.resample_batched(w, Nf, streams)
    else:
        out, U, W = drs.resample_batched(w, Nf, streams, return_uniforms=True, return_tables=True)
        np.testing.assert_array_equal(W, Wo)
        np.testing.assert_array_equal(U, Uo)
    np.testing.assert_array_equal(out, eo)


def test_batched_device_streams_advance(drs, orc):
    """BatchedStreams: positions advance on the device; two calls equal two
    host-stream calls; CUDA-graph replay draws fresh uniforms."""
    rng = np.random.default_rng(4)
    B, Mf, Nf = 150, 4096, 100
    w = np.exp(rng.standard_normal((B, Mf)))
    host = [drs.RngStream(5, (b,)) for b in range(B)]
    bs = drs.BatchedStreams([drs.RngStream(5, (b,)) for b in range(B)])
    wd = dev(w)
    for _ in range(2):
        e = drs.resample_batched(w, Nf, host)
        o = drs.resample_batched(wd, Nf, bs, check=False)
        np.testing.assert_array_equal(o.cpu().numpy(), e)
    assert (bs.positions() == 2 * (Nf + 1)).all()
    out = torch.empty((B, Nf), dtype=torch.int64, device="cuda")
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=side):
            r = drs.resample_batched(wd, Nf, bs, check=False)
    torch.cuda.current_stream().wait_stream(side)
    for _ in range(2):
        g.replay()
        torch.cuda.synchronize()
        e = drs.resample_batched(w, Nf, host)
        np.testing.assert_array_equal(r.cpu().numpy(), e)
    del out


def test_batched_invalid_weights_raise(drs):
    w = np.ones((10, 100))
    w[3, 5] = -1.0
    with pytest.raises(ValueError, match="invalid weight"):
        drs.resample_batched(w, 8, [drs.RngStream(1, (b,)) for b in range(10)])
    # a negative filter total (and NaN / inf totals): the search is skipped, no hang
    for bad in (-1.0, np.nan, np.inf):
        w = np.ones((300, 16384))
        w[7] = bad
        with pytest.raises(ValueError, match="invalid weight"):
            drs.resample_batched(w, 256, [drs.RngStream(2, (b,)) for b in range(300)])
    w = np.ones((10, 100))
    w[7] = 0.0
    with pytest.raises(ValueError, match="degenerate distribution"):
        drs.resample_batched(w, 8, [drs.RngStream(1, (b,)) for b in range(10)])


def _shard_emulation(orc, w, N, key, off, Gs, deferred=True):
    """The shard steps for G ranks run one after another on one GPU, with the
    all-gathers replaced by concatenation: the sharded table == the oracle's,
    every rank's U window == dr_sorted_uniforms bit for bit although each rank
    generated only its 1/G of the spacing tiles, the slices tile [0, N), and
    the indices == the oracle's DaC on the whole table."""
    from paper_2604_01356_b200.sharded import DeviceShardOps, ShardedWeightTable, slice_capacity

    ops = DeviceShardOps(deferred)
    M = w.size
    k0, k1 = key
    Uo, st_o = orc.sorted_uniforms(k0, k1, off, N)
    ts = ops.tile_size()
    nt = (N + 1 + ts - 1) // ts
    for G in Gs:
        parts = [dev(w[M * g // G: M * (g + 1) // G]) for g in range(G)]
        scans = [ops.shard_scan(p) for p in parts]
        totals = torch.cat([s[1] for s in scans])
        Wo, To, st = orc.build_table_sharded(w, G)
        np.testing.assert_array_equal(totals.cpu().numpy(), To)
        bounds = [nt * h // G for h in range(G + 1)]
        shares = [ops.unif_tile_totals((k0, k1), off, N, bounds[h], bounds[h + 1]) for h in range(G)]
        agg_all = torch.cat([a for a, _ in shares])
        zmin_all = torch.cat([z for _, z in shares])
        full = np.full(N, -1, dtype=np.int64)
        Ws, prev = [], 0
        for g in range(G):
            W, idx = ops.finalize(scans[g][0], totals, G, g)
            Ws.append(ops.materialize(W, idx).cpu().numpy())
            tab = ShardedWeightTable(W=W, index=idx, totals=totals, sizes=[p.numel() for p in parts], rank=g,
                                     world=G, totals_host=totals.cpu().tolist())
            ucap, ocap = slice_capacity(tab, N, ts)
            U, rngd, stg = ops.unif_local((k0, k1), off, N, agg_all, zmin_all, totals, G, g, ucap, ocap, False)
            a, b, ta, tb, ubase, obase, flags, _ = rngd.tolist()
            assert flags == 0 and int(stg.item()) & 0x600 == 0
            assert a == prev and ta * ts <= a and b <= min((tb + 1) * ts, N) and obase == a
            assert ubase == ta * ts - 1 and b - a <= ocap
            prev = b
            np.testing.assert_array_equal(U[a - ubase:b - ubase].cpu().numpy(), Uo[a:b])
            out = torch.empty(max(ocap, 1), dtype=torch.int64, device="cuda")
            ops.shard_match(tab, U, rngd, N, out)
            full[a:b] = out[: b - a].cpu().numpy()
            # the full-size re-run path gives the same slice
            U2, r2, _ = ops.unif_local((k0, k1), off, N, agg_all, zmin_all, totals, G, g, N + 1, N, True)
            assert r2.tolist()[:2] == [a, b] and r2.tolist()[4] == -1
            np.testing.assert_array_equal(U2[a + 1:b + 1].cpu().numpy(), Uo[a:b])
        assert prev == N
        np.testing.assert_array_equal(np.concatenate(Ws), Wo)
        np.testing.assert_array_equal(full, orc.match("dac", Wo, Uo))
    return st_o


@pytest.mark.parametrize("deferred", [True, False])
def test_sharded_single_gpu_emulation(drs, orc, deferred):
    rng = np.random.default_rng(1005)
    M, N = 1 << 20, (1 << 17) + 3
    w = np.exp(2 * rng.standard_normal(M))
    off = rng.integers(0, M - 1024)
    w[off:off + 1024] = (w.sum() - w[off:off + 1024].sum()) / 3 / 1024
    _shard_emulation(orc, w, N, orc.key_of(2005), 0, (1, 2, 4, 8), deferred)


def test_sharded_repair_at_rank_boundary(drs, orc):
    """A forced collapse of the sorted uniforms (a Philox draw above 1 - 2^-30
    at spacing i, found by scanning the stream: key (2005, (77,)), draw
    630216217) with the rank boundary placed just before it: the collapse sits
    in the first tiles of rank 1's window and the repair there must be exact
    (the previous version regenerated from the slice's own tile and could
    repair from an unrepaired value)."""
    N = 1 << 24
    key = orc.key_of(2005, (77,))
    for i in (3 * (1 << 22) + 7, 15 * (1 << 20) + 11):
        off = 630216217 - i
        Uo, st = orc.sorted_uniforms(key[0], key[1], off, N)
        assert st & 0x20  # the repair ran
        for lead in (1, 300, 700):
            M = 1 << 16
            w = np.random.default_rng(lead).random(M) + 0.5
            h = M // 2
            target = Uo[i - lead]  # rank 1's slice starts near u number i - lead
            w[:h] *= target / (1 - target) * w[h:].sum() / w[:h].sum()
            st_o = _shard_emulation(orc, w, N, key, off, (2,))
            assert st_o & 0x20


# ------------------------------------------------------------- fused sampler
@pytest.mark.parametrize("M,N", [(1 << 16, 1), (1 << 16, 1023), (1 << 20, 4095), (1 << 26, 1 << 16),
                                 (1 << 22, 150000), (3000000, 100001)])
def test_fused_dac_equals_two_pass_and_oracle(drs, orc, M, N):
    rng = np.random.default_rng(M ^ N)
    w = np.exp(4 * rng.standard_normal(M))
    w[rng.random(M) < 0.05] = 0.0
    t = drs.build_weight_table(w)
    fused = drs.dac_sampler(t, N, drs.RngStream(5, (N,)), mode="search", device=True)
    twopass = drs.dac_sampler(t, N, drs.RngStream(5, (N,)), mode="merge", device=True)
    np.testing.assert_array_equal(fused.cpu().numpy(), twopass.cpu().numpy())
    k0, k1 = orc.key_of(5, (N,))
    Uo, _ = orc.sorted_uniforms(k0, k1, 0, N)
    np.testing.assert_array_equal(fused.cpu().numpy(), orc.match("dac", t.cum, Uo))
    U = torch.empty(N, dtype=torch.float64, device="cuda")
    drs.dac_sampler(t, N, drs.RngStream(5, (N,)), mode="search", device=True, uniforms_out=U)
    np.testing.assert_array_equal(U.cpu().numpy(), Uo)


def test_fused_replay_and_repair(drs, orc, golden):
    W = golden[f"tbl_cum_{int(golden['tbl_count']) - 1}"]
    t = drs.WeightTable(W)
    for i in range(int(golden["rp_count"])):
        d = golden[f"rp_draws_{i}"]
        n = d.shape[0] - 1
        Uo, _ = orc.sorted_uniforms_from(d, n)
        for mode in ("search", "merge"):
            out = drs.dac_sampler(t, n, ReplayStream(d), mode=mode)
            np.testing.assert_array_equal(out, orc.match("dac", W, Uo))
    rng = np.random.default_rng(5)
    d = rng.random(50001)
    d[rng.random(50001) < 0.3] = 1 - 2.0 ** -53
    Uo, st = orc.sorted_uniforms_from(d, 50000)
    assert st & 0x20
    U = torch.empty(50000, dtype=torch.float64, device="cuda")
    out = drs.dac_sampler(t, 50000, ReplayStream(d), mode="search", uniforms_out=U)
    np.testing.assert_array_equal(U.cpu().numpy(), Uo)
    np.testing.assert_array_equal(out, orc.match("dac", W, Uo))


def test_device_stream_graph_replay(drs):
    w = np.exp(2 * np.random.default_rng(3).standard_normal(1 << 20))
    t = drs.build_weight_table(w)
    N = 4096
    for kind, kw in (("dac", {"mode": "search"}), ("dac", {"mode": "merge"}), ("ccf", {}), ("binary", {})):
        fn = {"dac": drs.dac_sampler, "ccf": drs.ccf_sampler, "binary": drs.binary_sampler}[kind]
        host = drs.RngStream(11)
        expect = [fn(t, N, host, **kw) for _ in range(3)]
        ds = drs.DeviceRngStream(11)
        out = torch.empty(N, dtype=torch.int64, device="cuda")
        extra = {} if kind == "binary" else {"uniforms_out": torch.empty(N, dtype=torch.float64, device="cuda")}
        fn(t, N, ds, device=True, out=out, **kw, **extra)  # warm (allocates workspaces)
        ds.offset_tensor.zero_()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            fn(t, N, ds, device=True, out=out, **kw, **extra)  # workspace for this stream
            ds.offset_tensor.zero_()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                fn(t, N, ds, device=True, out=out, **kw, **extra)
        torch.cuda.current_stream().wait_stream(s)
        ds.offset_tensor.zero_()
        got = []
        for _ in range(3):
            g.replay()
            got.append(out.cpu().numpy().copy())
        for a, b in zip(got, expect):
            np.testing.assert_array_equal(a, b)
        assert ds.position == host.position
