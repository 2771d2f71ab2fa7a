"""SURVEY 8(f)3 fused with the index writes: ``resample_and_gather`` /
``dr_sample_dac_gather`` must give exactly ``dac_sampler``'s indices (checked
against the oracle) and exactly ``states[idx // divisor]`` (numpy take), in
both the single-kernel regime (rows copied from the indices in registers) and
the two-pass pipeline (gather kernel after the match)."""

import numpy as np
import pytest
import torch

from oracle import oracle as orc

pytestmark = pytest.mark.gpu


def _oracle_dac(w, seed, n):
    W, _ = orc.build_table(w)
    k0, k1 = orc.key_of(seed)
    U, _ = orc.sorted_uniforms(k0, k1, 0, n)
    return orc.match("dac", W, U)


@pytest.mark.parametrize("M,N,d,div,mode", [
    (1 << 18, 1 << 10, 40, 1, "auto"),       # fused, EnGMF row width
    (1 << 20, 1 << 12, 40, 64, "auto"),      # fused, component -> particle
    (1 << 18, 1000, 3, 1, "search"),         # fused, ragged N, odd d (scalar lanes)
    (1 << 16, 1 << 16, 40, 1, "auto"),       # merge regime: two-pass + gather kernel
    (1 << 16, 777, 5, 16, "merge"),          # forced merge, ragged
    (1 << 22, 1 << 17, 4, 1, "search"),     # beyond the cooperative grid: two-pass
    (1, 9, 2, 1, "auto"),                    # one weight
])
def test_resample_and_gather_matches_sampler_then_take(drs, M, N, d, div, mode):
    rng = np.random.default_rng(M ^ N ^ d)
    w = np.exp(2.0 * rng.standard_normal(M))
    t = drs.build_weight_table(w)
    K = (M - 1) // div + 1
    states = rng.standard_normal((K, d))
    idx, rows = drs.resample_and_gather(t, N, drs.RngStream(4242), states, divisor=div, mode=mode)
    ref = drs.dac_sampler(t, N, drs.RngStream(4242), mode=mode)
    np.testing.assert_array_equal(idx, ref)
    if N <= 1 << 12:
        np.testing.assert_array_equal(idx, _oracle_dac(w, 4242, N))
    np.testing.assert_array_equal(rows, states[idx // div])


def test_resample_and_gather_device_stream_and_tensors(drs):
    rng = np.random.default_rng(11)
    M, N, d = 1 << 18, 2048, 40
    w = np.exp(rng.standard_normal(M))
    t = drs.build_weight_table(w)
    x = torch.from_numpy(rng.standard_normal((M, d))).cuda()
    ds = drs.DeviceRngStream(77)
    i1, r1 = drs.resample_and_gather(t, N, ds, x)
    i2, r2 = drs.resample_and_gather(t, N, ds, x)  # the device offset advanced by N + 1
    assert i1.is_cuda and r1.is_cuda and r1.shape == (N, d)
    hs = drs.RngStream(77)
    e1 = drs.dac_sampler(t, N, hs)
    e2 = drs.dac_sampler(t, N, hs)
    np.testing.assert_array_equal(i1.cpu().numpy(), e1)
    np.testing.assert_array_equal(i2.cpu().numpy(), e2)
    xs = x.cpu().numpy()
    np.testing.assert_array_equal(r2.cpu().numpy(), xs[e2])


def test_resample_and_gather_errors(drs):
    t = drs.build_weight_table(np.ones(100))
    with pytest.raises(IndexError):
        drs.resample_and_gather(t, 10, drs.RngStream(1), np.zeros((99, 2)))
    with pytest.raises(IndexError):
        drs.resample_and_gather(t, 10, drs.RngStream(1), np.zeros((9, 2)), divisor=11)
    with pytest.raises(ValueError):
        drs.resample_and_gather(t, 10, drs.RngStream(1), np.zeros((100, 2)), divisor=0)
    with pytest.raises(TypeError):
        drs.resample_and_gather(t, 10, object(), np.zeros((100, 2)))
    i, r = drs.resample_and_gather(t, 0, drs.RngStream(1), np.zeros((100, 3)))
    assert i.shape == (0,) and r.shape == (0, 3)
    # 10 // 10 = row 9 of 10 is the last one the sampler can reach
    i, r = drs.resample_and_gather(t, 50, drs.RngStream(1), np.arange(10.0), divisor=10)
    np.testing.assert_array_equal(r[:, 0], (i // 10).astype(np.float64))


@pytest.mark.parametrize("d", [1, 2, 7, 40, 129])
def test_gather_states_warp_blocks(drs, d):
    """k_gather_rows moves 64 rows per warp: ragged tails, odd and even row
    widths (scalar / 16-byte lanes), unsorted indices."""
    rng = np.random.default_rng(d)
    for K, N, div in [(1000, 64 * 37 + 5, 1), (300, 63, 4), (5000, 100_000, 1), (1, 65, 1)]:
        states = rng.standard_normal((K, d))
        idx = rng.integers(0, K * div, size=N)
        np.testing.assert_array_equal(drs.gather_states(states, idx, divisor=div), states[idx // div])


def test_gather_states_bad_index_leaves_other_rows(drs):
    """An index without a row (or a negative one) flags the status; the other
    rows of its warp block are still gathered (check=False exposes them)."""
    rng = np.random.default_rng(5)
    K, d = 100, 6
    states = torch.from_numpy(rng.standard_normal((K, d))).cuda()
    idx = torch.from_numpy(rng.integers(0, K, size=200)).cuda()
    for bad in (K, -1):
        j = idx.clone()
        j[70] = bad
        with pytest.raises(IndexError):
            drs.gather_states(states, j)
        out = drs.gather_states(states, j, check=False)
        keep = torch.ones(200, dtype=torch.bool, device="cuda")
        keep[70] = False
        assert torch.equal(out[keep], states[j[keep]])
