"""The single-pass (deferred-normalisation) table against the two-pass one.

``build_weight_table`` stores the in-tile chained sums L and the tile pairs
{C_g, D_t} (``dr_build_table_deferred``, include/drs.h); a search compares
S = C_g + (D_t + L) with a band around u T and forms fl(S / T) inside it, a
merge tile is turned into W (or W is formed at each probe).  These tests pin
(1) the deferred table's arrays bit for bit against the oracle twin
(``oracle.build_table_deferred``), (2) its cumulative weights against the
two-pass build and the oracle's W, and (3) every matcher and sampler on it
against the same call on the two-pass table, with uniforms placed exactly on,
one ulp below and one ulp above table values -- where the comparison must
agree with W < u (reference semantics: samplers.py:81-90, strict < lower bound).
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

EDGE_M = [1, 2, 15, 16, 17, 255, 256, 257, 8447, 8448, 8449, 32 * 8448, 32 * 8448 + 1, 3 * 8448 + 5,
          (1 << 18), (1 << 18) + 1, 33 * 8448 + 255, (1 << 20) + 7, 1000 * 8448 + 77]


def _weights(M, seed):
    rng = np.random.default_rng(seed)
    w = np.exp(4.0 * rng.standard_normal(M))
    w[rng.random(M) < 0.15] = 0.0
    if M > 40:
        w[8:40] = 0.0  # a zero run inside a level-1 block
    if w.sum() == 0:
        w[-1] = 1.0
    return w


def _boundary_u(W, rng, k=4000):
    """u on table values, one ulp either side, 1.0, the smallest positive."""
    pos = np.unique(rng.integers(0, W.size, size=min(k, W.size)))
    v = W[pos]
    u = np.concatenate([v, np.nextafter(v, 0.0), np.nextafter(v, 2.0), [1.0, 5e-324, 1e-300]])
    u = u[(u > 0.0) & (u <= 1.0)]
    return np.unique(u)


@pytest.mark.parametrize("M", EDGE_M)
def test_deferred_arrays_bit_exact_vs_oracle(drs, orc, M):
    w = _weights(M, M)
    t = drs.build_weight_table(w)
    assert t.deferred
    V, idx, W, st = orc.build_table_deferred(w)
    assert st == 0
    np.testing.assert_array_equal(t.device_values.cpu().numpy(), V)
    np.testing.assert_array_equal(t.device_index.cpu().numpy(), idx)
    np.testing.assert_array_equal(t.cum, W)
    t2 = drs.build_weight_table(w, deferred=False)
    assert not t2.deferred
    np.testing.assert_array_equal(t2.cum, W)
    ns = orc.search_entries(M)
    i2 = t2.device_index.cpu().numpy()
    np.testing.assert_array_equal(orc.index_l1_local(V, i2)[0][:ns], idx[:ns])
    np.testing.assert_array_equal(t2.device_index.cpu().numpy()[ns:], 0.0)  # direct header


@pytest.mark.parametrize("M", [(1 << 18) + 1, 300000, 64 * 8448, (1 << 22) + 5, 4097 * 8448])
def test_table_tail_equals_chain_and_levels(drs, M, monkeypatch):
    """dr_build_table_deferred finishes tables of 2^18 < M <= 16384 tiles with ONE
    launch after the pass (k_table_tail: every CTA folds the tile chain itself);
    DRS_NO_TABLE_TAIL=1 selects the chain + levels kernels it replaces (larger
    tables always use them).  Same association, same bytes."""
    w = torch.from_numpy(_weights(M, M + 1)).cuda()
    monkeypatch.delenv("DRS_NO_TABLE_TAIL", raising=False)
    a = drs.build_weight_table(w)
    monkeypatch.setenv("DRS_NO_TABLE_TAIL", "1")
    b = drs.build_weight_table(w)
    assert torch.equal(a.device_values.view(torch.int64), b.device_values.view(torch.int64))
    assert torch.equal(a.device_index.view(torch.int64), b.device_index.view(torch.int64))


@pytest.mark.parametrize("M", [17, 8449, 300_001, 256 * 8448 + 5])
def test_deferred_log_table_bit_exact(drs, orc, M):
    rng = np.random.default_rng(M)
    lw = 3.0 * rng.standard_normal(M)
    t = drs.build_weight_table_from_log(lw)
    assert t.deferred
    V, idx, W, st = orc.build_table_deferred(orc.exp(lw - lw.max()))
    np.testing.assert_array_equal(t.device_values.cpu().numpy(), V)
    np.testing.assert_array_equal(t.device_index.cpu().numpy(), idx)
    Wo, _ = orc.build_table_log(lw)
    np.testing.assert_array_equal(t.cum, Wo)
    np.testing.assert_array_equal(drs.build_weight_table_from_log(lw, deferred=False).cum, Wo)


@pytest.mark.parametrize("M", EDGE_M + [1 << 22])
def test_matchers_deferred_equal_direct_at_boundaries(drs, orc, M):
    w = _weights(M, 7 * M + 1)
    td = drs.build_weight_table(w)
    tt = drs.build_weight_table(w, deferred=False)
    W = tt.cum
    u = _boundary_u(W, np.random.default_rng(M))
    expect = orc.match("ccf", W, u)
    for mode in ("auto", "merge", "search"):
        a = drs.dac_match(u, td, mode=mode)
        np.testing.assert_array_equal(a, expect, err_msg=f"dac {mode} M={M}")
        np.testing.assert_array_equal(drs.dac_match(u, tt, mode=mode), expect)
    np.testing.assert_array_equal(drs.ccf_match(u, td), expect)
    # unsorted u through the binary matcher (duplicates and u = 1 included)
    ub = np.random.default_rng(3).permutation(np.concatenate([u, u[: len(u) // 3]]))
    from paper_2604_01356_b200 import samplers

    ud = torch.from_numpy(ub).cuda()
    np.testing.assert_array_equal(samplers._lower_bounds(td, ud).cpu().numpy(), orc.match("binary", W, ub))


def test_matchers_deferred_out_of_range_u(drs, orc):
    """check=False lets u outside (0, 1] through: the deferred key maps them
    like the direct comparison (u <= 0 -> index 0, u > 1 -> M-1)."""
    w = _weights(5000, 11)
    td = drs.build_weight_table(w)
    tt = drs.build_weight_table(w, deferred=False)
    u = np.array([-1.0, -0.0, 0.0, 0.25, 0.5, 1.0, 1.0 + 2**-52, 7.0, np.inf])
    for mode in ("merge", "search"):
        np.testing.assert_array_equal(drs.dac_match(u, td, check=False, mode=mode),
                                      drs.dac_match(u, tt, check=False, mode=mode))
    np.testing.assert_array_equal(drs.ccf_match(u, td, check=False), drs.ccf_match(u, tt, check=False))


@pytest.mark.parametrize("M,N", [(65536, 1024), (1 << 20, 1 << 20), (1 << 22, 1 << 16), (3 * 8448 + 5, 4000)])
def test_samplers_deferred_equal_direct(drs, M, N):
    w = _weights(M, M + N)
    td = drs.build_weight_table(w)
    tt = drs.build_weight_table(w, deferred=False)
    for fn in (drs.dac_sampler, drs.ccf_sampler, drs.binary_sampler):
        a = fn(td, N, drs.RngStream(99))
        b = fn(tt, N, drs.RngStream(99))
        np.testing.assert_array_equal(a, b, err_msg=fn.__name__)
    for mode in ("merge", "search"):
        np.testing.assert_array_equal(drs.dac_sampler(td, N, drs.RngStream(5), mode=mode),
                                      drs.dac_sampler(tt, N, drs.RngStream(5), mode=mode))


def test_gather_fused_on_deferred(drs):
    M, N, d = 1 << 18, 1 << 12, 6
    w = _weights(M, 3)
    td = drs.build_weight_table(w)
    tt = drs.build_weight_table(w, deferred=False)
    states = torch.randn(M, d, dtype=torch.float64, device="cuda")
    ia, ga = drs.resample_and_gather(td, N, drs.RngStream(8), states)
    ib, gb = drs.resample_and_gather(tt, N, drs.RngStream(8), states)
    assert torch.equal(torch.as_tensor(ia).cpu(), torch.as_tensor(ib).cpu())
    assert torch.equal(ga, gb)


def test_verification_on_deferred(drs):
    w = _weights(70_000, 12)
    td = drs.build_weight_table(w)
    tt = drs.build_weight_table(w, deferred=False)
    np.testing.assert_array_equal(td.weights(), tt.weights())
    for x, lo, hi in ((0.3, 0, 69_999), (1.0, 10, 500), (0.0, 0, 69_999)):
        assert drs.upper_bound_search(td, lo, hi, x) == drs.upper_bound_search(tt, lo, hi, x)
    st_a, st_b = drs.OpStats(), drs.OpStats()
    drs.dac_sampler(td, 3000, drs.RngStream(4), stats=st_a)
    drs.dac_sampler(tt, 3000, drs.RngStream(4), stats=st_b)
    assert st_a == st_b


def test_deferred_table_errors(drs):
    with pytest.raises(ValueError, match="degenerate distribution"):
        drs.build_weight_table([0.0, 0.0])
    for bad in ([-1.0, 2.0], [np.nan], [np.inf, 1.0]):
        with pytest.raises(ValueError, match="invalid weight"):
            drs.build_weight_table(bad)
    with pytest.raises(ValueError, match="accumulation overflow"):
        drs.build_weight_table([1e308, 1e308])


@pytest.mark.parametrize("M,G", [(20, 3), (300_001, 3), ((1 << 20) + 5, 4)])
def test_sharded_deferred_shards(drs, orc, M, G):
    """The single-pass shard build (dr_shard_scan_deferred + _finalize_deferred,
    header mode 2: S = O_g + (C + (D + L))): every shard's W == the oracle's
    sharded table, its index == the index of that W, and the matchers on the
    shard's values agree with the oracle on u's placed on its W values."""
    from paper_2604_01356_b200.cdf import WeightTable
    from paper_2604_01356_b200.sharded import DeviceShardOps

    ops = DeviceShardOps()
    w = _weights(M, M + G)
    cuts = [M * g // G for g in range(G + 1)]
    scans = [ops.shard_scan(torch.from_numpy(w[cuts[g]:cuts[g + 1]]).cuda()) for g in range(G)]
    totals = torch.cat([s[1] for s in scans])
    Wo, To, st = orc.build_table_sharded(w, G)
    np.testing.assert_array_equal(totals.cpu().numpy(), To)
    for g in range(G):
        V, idx = ops.finalize(scans[g][0], totals, G, g)
        Wg = Wo[cuts[g]:cuts[g + 1]]
        np.testing.assert_array_equal(ops.materialize(V, idx).cpu().numpy(), Wg)
        ns = orc.search_entries(Wg.size)
        ref_idx, _ = orc.index_l1_local(V.cpu().numpy(), orc.build_index(Wg))
        np.testing.assert_array_equal(idx.cpu().numpy()[:ns], ref_idx[:ns])
        t = WeightTable(None, _built=(V, idx, True))
        u = _boundary_u(Wg, np.random.default_rng(g))
        u = u[u <= Wg[-1]]
        expect = orc.match("ccf", Wg, u)
        for mode in ("merge", "search"):
            np.testing.assert_array_equal(drs.dac_match(u, t, mode=mode), expect)
        np.testing.assert_array_equal(drs.ccf_match(u, t), expect)
