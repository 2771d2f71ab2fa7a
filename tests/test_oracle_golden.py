"""The CPU oracle pinned against the reference's own outputs (tests/golden).

CPU only.  These tests make the oracle trustworthy as the checker for the
GPU parity tests: the drs_port_* functions must reproduce the reference bit
for bit, and the drs_ref_* functions (device association) must agree with
the reference up to fp64 scan reassociation.
"""

import hashlib

import numpy as np
import pytest

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


def test_philox_matches_numpy(orc):
    for seed, key, off, k in [(2003, (), 0, 37), (7, (3, 1), 5, 64), (0, (), 1001, 9)]:
        k0, k1 = orc.key_of(seed, key)
        gen = np.random.Generator(np.random.Philox(np.random.SeedSequence(seed, spawn_key=key)))
        if off:
            gen.random(off)
        np.testing.assert_array_equal(orc.uniforms(k0, k1, off, k), gen.random(k))


def test_log_within_one_ulp_of_numpy(orc):
    rng = np.random.default_rng(0)
    x = np.concatenate([rng.random(20000), np.exp(-700 * rng.random(2000)), rng.random(200) * 1e-310,
                        [1.0, 0.5, 2.0 ** -53, 2.0 ** -54, 1 - 2.0 ** -53]])
    d = ulps(orc.log(x), np.log(x))
    assert d.max() <= 1
    assert (d > 0).mean() < 0.02


def test_port_build_table_is_bit_exact(orc, golden):
    for i in range(int(golden["tbl_count"])):
        W, st = orc.port_build_table(golden[f"tbl_raw_{i}"])
        assert st == 0
        np.testing.assert_array_equal(W, golden[f"tbl_cum_{i}"])


def test_device_association_table_close_to_reference(orc, golden):
    for i in range(int(golden["tbl_count"])):
        raw, ref = golden[f"tbl_raw_{i}"], golden[f"tbl_cum_{i}"]
        W, st = orc.build_table(raw)
        assert st == 0 and W[-1] == 1.0
        assert np.all(np.diff(W) >= 0.0)
        # reassociation drift only; measured max well below 1e4 ulp
        assert np.abs(W - ref).max() <= 1e-12


def test_kat_tables(orc):
    W, st = orc.build_table([2.0, 1.0, 1.0])
    np.testing.assert_array_equal(W, [0.5, 0.75, 1.0])
    W, st = orc.build_table([1.0])
    np.testing.assert_array_equal(W, [1.0])
    W, st = orc.build_table([1.0, 0.0, 0.0])
    np.testing.assert_array_equal(W, [1.0, 1.0, 1.0])
    assert orc.build_table([1e308, 1e308])[1] & 0x4
    assert orc.build_table([0.0, 0.0])[1] & 0x2
    assert orc.build_table([-1.0, 2.0])[1] & 0x1
    assert orc.build_table([np.nan])[1] & 0x1


def test_port_matchers_equal_reference_cases(orc, golden):
    n = 0
    for W, u, e in golden_cases(golden):
        for kind in ("binary", "ccf", "dac"):
            np.testing.assert_array_equal(orc.match(kind, W, u), e)
        n += 1
    assert n == 300


def test_exhaustive_tables_digest(orc, golden):
    h = hashlib.sha256()
    count = 0
    for raw in enumerate_weight_tables(8):
        W, st = orc.port_build_table(raw)
        np.testing.assert_array_equal(W, reference_table_exact(raw)) if count % 997 == 0 else None
        u = boundary_query_set(W)
        e = orc.match("dac", W, u)
        h.update(W.tobytes())
        h.update(u.tobytes())
        h.update(e.astype(np.int64).tobytes())
        count += 1
    assert count == int(golden["exh_count"])
    assert h.digest() == golden["exh_digest"].tobytes()


def test_exhaustive_tables_device_association(orc):
    # the device association on small-integer weights is exact too
    for raw in enumerate_weight_tables(6):
        W, _ = orc.build_table(raw)
        np.testing.assert_array_equal(W, reference_table_exact(raw))
        u = boundary_query_set(W)
        np.testing.assert_array_equal(orc.match("dac", W, u), linear_scan_bulk(W, u))


def test_port_sorted_uniforms_bit_exact_with_numpy_log(orc, golden):
    # same draws, np.log spacings: the port's sequential association is the reference's
    for i, (seed, n) in enumerate(golden["su_cases"]):
        d = PhiloxStream(int(seed)).uniforms(int(n) + 1)
        U, _ = orc.sorted_from_z(-np.log(d), int(n), association="port")
        np.testing.assert_array_equal(U, golden[f"su_U_{i}"])


def test_device_association_sorted_uniforms_close(orc, golden):
    for i, (seed, n) in enumerate(golden["su_cases"]):
        k0, k1 = orc.key_of(int(seed))
        U, _ = orc.sorted_uniforms(k0, k1, 0, int(n))
        ref = golden[f"su_U_{i}"]
        assert np.all(np.diff(U) > 0) and U[0] > 0 and U[-1] < 1
        assert np.abs(U - ref).max() <= 1e-13


def test_replay_and_repair_cases(orc, golden):
    for i in range(int(golden["rp_count"])):
        d = golden[f"rp_draws_{i}"]
        n = d.shape[0] - 1
        ref = golden[f"rp_U_{i}"]
        # port with numpy's log is the reference exactly
        U, _ = orc.sorted_from_z(-np.log(d), n, association="port")
        np.testing.assert_array_equal(U, ref)
        # device association: strictly increasing inside (0, 1), close to the reference
        U2, _ = orc.sorted_uniforms_from(d, n)
        assert U2[0] > 0 and U2[-1] < 1 and np.all(np.diff(U2) > 0)
        assert np.abs(U2 - ref).max() <= 1e-12
    np.testing.assert_array_equal(orc.repair_open_strict(golden["repair_in"]), golden["repair_out"])


def test_stubbed_halves_kat(orc):
    U, _ = orc.sorted_uniforms_from([0.5, 0.5, 0.5], 2)
    np.testing.assert_allclose(U, [1 / 3, 2 / 3], rtol=1e-15)


def test_c1_port_samplers_match_reference(orc, golden):
    W, _ = orc.port_build_table(golden[f"tbl_raw_{int(golden['tbl_count']) - 1}"])
    # reference sorted_uniforms on numpy Philox draws, then the port's matchers
    d = PhiloxStream(2001).uniforms(1025)
    U, _ = orc.sorted_from_z(-np.log(d), 1024, association="port")
    np.testing.assert_array_equal(orc.match("dac", W, U), golden["c1_dac"])
    np.testing.assert_array_equal(orc.match("ccf", W, U), golden["c1_ccf"])
    np.testing.assert_array_equal(orc.match("binary", W, d[:1024]), golden["c1_binary"])


def test_port_sampler_uses_port_association(orc):
    W, _ = orc.port_build_table(np.exp(np.random.default_rng(3).standard_normal(5000)))
    k0, k1 = orc.key_of(42)
    out = orc.port_sampler("dac", W, k0, k1, 0, 300)
    U, _ = orc.port_sorted_uniforms(k0, k1, 0, 300)
    np.testing.assert_array_equal(out, linear_scan_bulk(W, U))
    np.testing.assert_array_equal(orc.port_sampler("ccf", W, k0, k1, 0, 300), out)


def test_index_layout(orc):
    W, _ = orc.build_table(np.random.default_rng(1).random(1000))
    idx = orc.build_index(W)
    # level 1: last entry of every 16-block, padded with +inf to a multiple of 16
    n1 = -(-1000 // 16)
    np.testing.assert_array_equal(idx[:n1], W[np.minimum(np.arange(1, n1 + 1) * 16 - 1, 999)])
    assert np.all(np.isinf(idx[n1:64]))
    n2 = -(-n1 // 16)
    np.testing.assert_array_equal(idx[64:64 + n2], W[np.minimum(np.arange(1, n2 + 1) * 256 - 1, 999)])


def test_sharded_association_consistent(orc):
    rng = np.random.default_rng(9)
    w = np.exp(2 * rng.standard_normal(50000))
    w[rng.random(50000) < 0.1] = 0
    for G in (1, 2, 3, 8):
        W, T, st = orc.build_table_sharded(w, G)
        assert st == 0 and W[-1] == 1.0 and np.all(np.diff(W) >= 0)
        # the boundary value of shard g equals the last W of shard g-1
        O = 0.0
        Tt = 0.0
        for t in T:
            Tt = Tt + t
        for g in range(G):
            a = 50000 * g // G
            if g:
                assert W[a - 1] == min(O / Tt, 1.0)
            O = O + T[g]
    W1, _, _ = orc.build_table_sharded(w, 1)
    np.testing.assert_array_equal(W1, orc.build_table(w)[0])


def test_batched_oracle_equals_per_filter(orc):
    rng = np.random.default_rng(4)
    B, Mf, Nf = 5, 3000, 40
    w = rng.random((B, Mf))
    keys = np.array([list(orc.key_of(100 + b)) + [b * 7] for b in range(B)], dtype=np.uint64)
    out, U, W, st = orc.resample_batched(w, Nf, keys)
    assert st & ~0x20 == 0
    for b in range(B):
        Wb, _ = orc.build_table(w[b])
        np.testing.assert_array_equal(W[b], Wb)
        Ub, _ = orc.sorted_uniforms(int(keys[b, 0]), int(keys[b, 1]), int(keys[b, 2]), Nf)
        np.testing.assert_array_equal(U[b], Ub)
        np.testing.assert_array_equal(out[b], linear_scan_bulk(Wb, Ub))


@pytest.mark.parametrize("n", [1, 2, 1023, 1024, 1025, 4096])
def test_chain_scan_tile_edges(orc, n):
    x = np.random.default_rng(n).random(n)
    for K in (4, 33):
        S, tot = orc.chain_scan(x, K)
        assert np.all(np.diff(S) >= 0)
        assert tot == S[-1]
        assert np.abs(S - np.cumsum(x)).max() <= 1e-12 * n


@pytest.mark.parametrize("K", [4, 33])
def test_chain_scan_group_boundaries_monotone(orc, K):
    """Across groups of 32 tiles: S non-decreasing, S[-1] == total, zero runs
    at the tile and group edges stay flat (no 1-ulp dips), drift small."""
    tile = 256 * K
    n = 600 * tile + 17
    rng = np.random.default_rng(K)
    x = np.exp(3 * rng.standard_normal(n))
    for e in (31 * tile, 32 * tile, 64 * tile, 512 * tile):
        x[e - 50:e + 50] = 0.0
    S, tot = orc.chain_scan(x, K)
    assert np.all(np.diff(S) >= 0)
    assert tot == S[-1]
    ref = np.cumsum(x)
    assert np.abs(S - ref).max() <= 1e-12 * ref[-1]


def test_device_exp_twin_within_one_ulp(orc):
    """oracle/drs_ref_exp (the device exp's twin): <= 1 ulp from np.exp and
    < 1 ulp from an extended-precision exp over the whole finite range."""
    rng = np.random.default_rng(5)
    x = np.concatenate([rng.uniform(-745.0, 709.7, 400_000), rng.uniform(-1, 1, 100_000),
                        -rng.exponential(40.0, 100_000), [0.0, -0.0, 709.78, -745.13, -708.4, -1e-300]])
    y = orc.exp(x)
    npy = np.exp(x)
    normal = npy >= np.finfo(float).tiny
    assert np.all(np.abs(y[normal] - npy[normal]) <= np.spacing(npy[normal]))
    assert np.all(np.abs(y[~normal] - npy[~normal]) <= 5e-324)
    ref = np.exp(x.astype(np.longdouble))
    err = np.abs((y.astype(np.longdouble) - ref) / np.spacing(npy).astype(np.longdouble))
    assert float(err[normal].max()) < 1.0
    assert np.isnan(orc.exp(np.array([np.nan]))[0]) and orc.exp(np.array([800.0]))[0] == np.inf
    assert orc.exp(np.array([-800.0]))[0] == 0.0


def test_log_table_close_to_reference_pipeline(orc):
    """build_table_log == build_table(exp(lw - max)) with the device exp; and
    within the association drift of the reference's np.exp + build_weight_table."""
    rng = np.random.default_rng(6)
    for M in (1, 17, 8449, 300_000):
        lw = -0.5 * rng.chisquare(6, size=M) + np.log(rng.dirichlet(np.ones(M))) if M > 1 else np.array([3.0])
        W, st = orc.build_table_log(lw)
        assert st == 0 and W[-1] == 1.0 and np.all(np.diff(W) >= 0)
        Wd, _ = orc.build_table(orc.exp(lw - lw.max()))
        np.testing.assert_array_equal(W, Wd)
        Wp, _ = orc.port_build_table(np.exp(lw - lw.max()))
        assert np.abs(W - Wp).max() <= 1e-12
    _, st = orc.build_table_log(np.array([0.0, np.nan, 1.0]))
    assert st & 0x1
