"""The per-call host path of the samplers (drs_host.c, dr_sample_dac_sync):
a host-result call (a RngStream, no out= / uniforms_out= / stats=) goes
through the CPython extension and, for dac in the single-kernel regime,
through the cached one-node graph launch.  Its indices must equal the
device path's and the oracle's for the same stream positions, with the
graph re-parameterised every call (stream offsets, result buffers) and
rebuilt when the grid changes."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def test_extension_loaded(drs):
    from paper_2604_01356_b200 import samplers

    assert samplers._hc is not None, "_drshost.so is not built (make -C paper_2604_01356_b200/csrc)"


@pytest.mark.parametrize("kind", ["dac", "ccf"])
def test_host_path_equals_device_path(drs, kind):
    fn = {"dac": drs.dac_sampler, "ccf": drs.ccf_sampler}[kind]
    rng = np.random.default_rng(77)
    table = drs.build_weight_table(np.exp(3.0 * rng.standard_normal(1 << 18)), deferred=False)
    # n changes the fused grid (n + 1 <= 512 x 148), and the last one leaves the single-kernel regime
    for n in (1, 1023, 5000, 1 << 14, 5000, 70000, 1 << 17):
        s_host, s_dev = drs.RngStream(9, (n,)), drs.RngStream(9, (n,))
        for rep in range(3):
            h = fn(table, n, s_host)
            d = fn(table, n, s_dev, device=True).cpu().numpy()
            assert isinstance(h, np.ndarray) and h.dtype == np.int64 and h.shape == (n,)
            assert np.array_equal(h, d), (kind, n, rep)
            assert s_host.draws == s_dev.draws == (rep + 1) * (n + 1)


def test_host_path_matches_oracle(drs):
    from oracle import oracle as orc

    rng = np.random.default_rng(78)
    w = np.exp(rng.standard_normal(1 << 16))
    table = drs.build_weight_table(w)
    W = table.cum
    s = drs.RngStream(31)
    k0, k1 = orc.key_of(31)
    pos = 0
    for n in (4096, 65535, 4096):
        out = drs.dac_sampler(table, n, s)
        U, _ = orc.sorted_uniforms(k0, k1, pos, n)
        pos += n + 1
        assert np.array_equal(out, orc.match("dac", W, U)), n


def test_host_path_on_a_side_stream(drs):
    """the plan and the graph are per (device, stream)"""
    table = drs.build_weight_table(np.arange(1.0, 5001.0))
    ref = drs.dac_sampler(table, 3000, drs.RngStream(5))
    side = torch.cuda.Stream()
    with torch.cuda.stream(side):
        got = drs.dac_sampler(table, 3000, drs.RngStream(5))
    assert np.array_equal(ref, got)
