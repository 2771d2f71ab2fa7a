"""the edge-case contract of the reference's public API,
checked through the GPU package (names, messages, dtypes and draw accounting
as in samplers.py / cdf.py / randkit.py)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _samplers(drs):
    return {"dac": drs.dac_sampler, "ccf": drs.ccf_sampler, "binary": drs.binary_sampler}


def test_n_zero_returns_empty_and_draws_nothing(drs):
    """samplers.py:241-244, randkit.py:82-83"""
    t = drs.build_weight_table([1.0, 2.0, 3.0])
    for name, fn in _samplers(drs).items():
        s = drs.RngStream(1)
        out = fn(t, 0, s)
        assert isinstance(out, np.ndarray) and out.dtype == np.int64 and out.shape == (0,), name
        assert s.draws == 0, name
    s = drs.RngStream(1)
    u = drs.sorted_uniforms(s, 0)
    assert u.shape == (0,) and u.dtype == np.float64 and s.draws == 0


def test_draw_accounting(drs):
    """n + 1 draws per sorted_uniforms / sorted sampler, n per binary_sampler (test_randkit.py:60-65)"""
    t = drs.build_weight_table([1.0, 2.0, 3.0])
    for name, fn in _samplers(drs).items():
        s = drs.RngStream(2)
        fn(t, 10, s)
        assert s.draws == (10 if name == "binary" else 11), name


def test_empty_u_to_matchers(drs):
    """samplers.py:70-71, 173-174, 204-205"""
    t = drs.build_weight_table([1.0, 1.0])
    for fn in (drs.ccf_match, drs.dac_match):
        out = fn(np.zeros(0), t)
        assert out.dtype == np.int64 and out.shape == (0,)


def test_negative_n(drs):
    """randkit.py:80-81"""
    with pytest.raises(ValueError, match="n must be >= 0"):
        drs.sorted_uniforms(drs.RngStream(0), -1)
    t = drs.build_weight_table([1.0])
    for fn in (drs.dac_sampler, drs.ccf_sampler):
        with pytest.raises(ValueError, match="n must be >= 0"):
            fn(t, -1, drs.RngStream(0))


@pytest.mark.parametrize("raw", [[], np.zeros((2, 3)), np.zeros((0,))])
def test_empty_or_2d_weights(drs, raw):
    """cdf.py:72-73: the same message for a 2-D array"""
    with pytest.raises(ValueError, match="empty distribution"):
        drs.build_weight_table(raw)


def test_trailing_and_leading_zero_weights(drs):
    """cdf.py:85-88 and the lower-bound tie rule samplers.py:86; SPEC.md:118"""
    t = drs.build_weight_table([1.0, 0.0, 0.0])
    np.testing.assert_array_equal(t.cum, [1.0, 1.0, 1.0])
    np.testing.assert_array_equal(drs.dac_match([1.0], t), [0])
    np.testing.assert_array_equal(drs.ccf_match([1.0], t), [0])
    t = drs.build_weight_table([0.0, 1.0])
    np.testing.assert_array_equal(t.cum, [0.0, 1.0])
    for fn in _samplers(drs).values():
        assert np.all(fn(t, 1000, drs.RngStream(3)) == 1)


def test_u_equal_one_maps_to_first_full_index(drs):
    """SPEC.md:221, cdf.py:88"""
    t = drs.build_weight_table([1.0, 2.0, 0.0, 0.0])
    for fn in (drs.ccf_match, drs.dac_match):
        np.testing.assert_array_equal(fn([0.5, 1.0], t), [1, 1])
    assert drs.linear_oracle(t, 1.0) == 1


def test_duplicate_u_check_and_no_check(drs):
    """samplers.py:74-75 (check=True) versus the sampler path (check=False)"""
    t = drs.build_weight_table([1.0, 1.0, 1.0])
    u = [0.2, 0.5, 0.5, 0.9]
    for fn in (drs.ccf_match, drs.dac_match):
        with pytest.raises(ValueError, match="input not sorted"):
            fn(u, t)
        np.testing.assert_array_equal(fn(u, t, check=False), [0, 1, 1, 2])


def test_out_of_support_u(drs):
    """samplers.py:72-73, 57"""
    t = drs.build_weight_table([1.0, 1.0])
    for fn in (drs.ccf_match, drs.dac_match):
        with pytest.raises(ValueError, match=r"uniforms must lie in \(0, 1\]"):
            fn([0.0, 0.5], t)
        with pytest.raises(ValueError, match=r"uniforms must lie in \(0, 1\]"):
            fn([0.5, 1.5], t)
    for bad in (0.0, 1.5, -1.0):
        with pytest.raises(ValueError, match=r"u must lie in \(0, 1\]"):
            drs.linear_oracle(t, bad)


def test_array_like_inputs(drs):
    """cdf.py:71, samplers.py:168,199: lists are coerced to contiguous float64"""
    t = drs.build_weight_table([2, 1, 1])  # ints
    np.testing.assert_array_equal(t.cum, [0.5, 0.75, 1.0])
    np.testing.assert_array_equal(drs.dac_match([0.1, 0.6, 0.8], drs.WeightTable([0.25, 0.5, 0.75, 1.0])), [0, 2, 3])


def test_weight_table_top_entry(drs):
    """cdf.py:39-40"""
    with pytest.raises(ValueError, match="cumulative weights must end at exactly 1"):
        drs.WeightTable([0.5, 0.9])
    with pytest.raises(ValueError, match="cumulative weights must be non-decreasing from >= 0"):
        drs.WeightTable([0.5, 0.4, 1.0])
    assert drs.build_weight_table(np.exp(np.random.default_rng(0).standard_normal(1000))).cum[-1] == 1.0


def test_output_dtype_and_order(drs):
    """samplers.py:172,203,242; int64, matchers and sorted
    samplers non-decreasing, binary_sampler in draw order"""
    t = drs.build_weight_table(np.exp(np.random.default_rng(1).standard_normal(5000)))
    for name, fn in _samplers(drs).items():
        out = fn(t, 4000, drs.RngStream(9))
        assert out.dtype == np.int64 and out.min() >= 0 and out.max() < 5000
        if name != "binary":
            assert np.all(np.diff(out) >= 0), name
    b = drs.binary_sampler(t, 4000, drs.RngStream(9))
    assert not np.all(np.diff(b) >= 0)  # draw order, not sorted


def test_upper_bound_search_errors(drs):
    """cdf.py:103-107"""
    t = drs.build_weight_table([1.0, 1.0, 1.0])
    with pytest.raises(ValueError, match="empty range"):
        drs.upper_bound_search(t, 2, 1, 0.5)
    with pytest.raises(IndexError):
        drs.upper_bound_search(t, 0, 3, 0.5)
    assert drs.upper_bound_search(t, 0, 2, 0.5) == 1


def test_stats_counted_on_device(drs):
    """stats= is the reference's instrumented count (test_samplers.py:174-188
    shape): binary / ccf never nest scopes, dac never exceeds its budgets."""
    t = drs.build_weight_table([1.0, 1.0, 1.0, 1.0])
    s = drs.OpStats()
    drs.binary_sampler(t, 100, drs.RngStream(1), stats=s)
    assert s.max_depth == 0 and 0 < s.probes <= 100 * 3
    s = drs.OpStats()
    drs.ccf_sampler(t, 100, drs.RngStream(1), stats=s)
    assert s.max_depth == 0 and 100 <= s.comparisons <= 2 * 100 + 100
    s = drs.OpStats()
    drs.ccf_match([0.5], t, stats=s)
    assert (s.comparisons, s.probes) == (2, 0)  # the cursor stops on W[1] = 0.5
    s = drs.OpStats()
    drs.dac_sampler(t, 4, drs.RngStream(0), stats=s)
    assert 1 <= s.max_depth <= 3 and s.probes <= 4 * 3
    s = drs.OpStats()
    assert drs.dac_match(np.empty(0), t, stats=s).shape == (0,) and s == drs.OpStats()


def test_device_in_device_out(drs):
    t = drs.build_weight_table(torch.rand(100, dtype=torch.float64, device="cuda") + 0.1)
    u = torch.sort(torch.rand(50, dtype=torch.float64, device="cuda"))[0]
    out = drs.dac_match(u, t)
    assert isinstance(out, torch.Tensor) and out.is_cuda and out.dtype == torch.int64
    out = drs.dac_sampler(t, 50, drs.RngStream(1), device=True)
    assert isinstance(out, torch.Tensor) and out.is_cuda


def test_out_buffers_validated(drs):
    """out= / uniforms_out= must be contiguous tensors of the right dtype and
    length on the current device (or device-accessible pinned memory): a bad
    buffer raises instead of being written out of bounds."""
    t = drs.build_weight_table([1.0, 2.0, 3.0])
    n = 64
    with pytest.raises(ValueError, match="dtype"):
        drs.dac_sampler(t, n, drs.RngStream(1), out=torch.empty(n, dtype=torch.int32, device="cuda"))
    with pytest.raises(ValueError, match="elements"):
        drs.dac_sampler(t, n, drs.RngStream(1), out=torch.empty(n - 1, dtype=torch.int64, device="cuda"))
    with pytest.raises(ValueError, match="contiguous"):
        drs.ccf_sampler(t, n, drs.RngStream(1), out=torch.empty(2 * n, dtype=torch.int64, device="cuda")[::2])
    with pytest.raises(ValueError, match="pinned"):
        drs.binary_sampler(t, n, drs.RngStream(1), out=torch.empty(n, dtype=torch.int64))
    with pytest.raises(ValueError, match="dtype"):
        drs.dac_sampler(t, n, drs.RngStream(1), uniforms_out=torch.empty(n, dtype=torch.float32, device="cuda"))
    with pytest.raises(TypeError):
        drs.dac_sampler(t, n, drs.RngStream(1), out=np.empty(n, dtype=np.int64))
    # pinned host buffers are written directly
    out = torch.empty(n, dtype=torch.int64, pin_memory=True)
    res = drs.dac_sampler(t, n, drs.RngStream(1), out=out, device=True)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(out.numpy(), drs.dac_sampler(t, n, drs.RngStream(1)))
    assert res.data_ptr() == out.data_ptr()


def test_opstats_small_shapes(drs):
    """Counts on the smallest shapes (values from the reference itself): one table entry (no probe ever), one u
    (the root scope only), u = 1 exactly, and device-tensor inputs."""
    one = drs.build_weight_table([5.0])
    s = drs.OpStats()
    drs.dac_match([0.3, 0.9, 1.0], one, stats=s)
    assert (s.comparisons, s.probes) == (0, 0) and s.max_depth == 1  # the root scope is filled
    t = drs.WeightTable([0.25, 0.5, 0.75, 1.0])
    s = drs.OpStats()
    drs.dac_match([0.6], t, stats=s)
    assert (s.probes, s.max_depth) == (2, 1)
    s = drs.OpStats()
    drs.ccf_match(torch.tensor([0.1, 1.0], dtype=torch.float64, device="cuda"), t, stats=s)
    assert s.comparisons == 3 + 2
    s = drs.OpStats()
    drs.binary_sampler(t, 3, __import__("tests.helpers", fromlist=["ReplayStream"]).ReplayStream([0.25, 0.5, 1.0]),
                       stats=s)
    assert s.probes == 6 and s.max_depth == 0
