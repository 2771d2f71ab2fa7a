"""Parity at every BASELINE config at full size -- config 5 (M = 2^30, N = 2^24), the
north star's device-mode boundary report at every config.

Config 5 is the box-scale case: an 8 GiB table with 8 index levels and byte
offsets above 2^32, a 25%-of-mass spike block (the long-run split of the
merge, ``k_merge_heavy``), and N = 2^24 sorted uniforms, where the
reference's exactness check (randkit.py:95-100) fires in most calls.

Exact mode: the reference's matchers (oracle port of samplers.py:93-146) on
the device's own W and U reproduce the device's indices bit for bit for dac
(auto = index search, merge), ccf and binary; W and U equal the oracle's
device-association twins bit for bit.  Device mode against the reference
association (oracle/parity.py): every index flip lies within the measured
W + U drift of a boundary.
"""

import numpy as np
import pytest
import torch

from tests.helpers import boundary_query_set, enumerate_weight_tables

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def c5():
    from bench import CONFIGS, make_weights

    w = make_weights("c5")
    return w, CONFIGS["c5"]


def test_c5_full_size_bit_exact(drs, orc, c5):
    from oracle import parity

    w, c = c5
    M, N = c["M"], c["N"]
    assert w.size == M
    t = drs.build_weight_table(w)
    W = t.cum
    Wo, st = orc.build_table(w)
    assert st == 0
    np.testing.assert_array_equal(W, Wo)  # K1 at 2^30: bit-exact vs the device-association twin
    del Wo
    assert W[-1] == 1.0
    k0, k1 = orc.key_of(c["useed"])
    Uo, _ = orc.sorted_uniforms(k0, k1, 0, N)
    Wref, _ = orc.port_build_table(w)
    U = torch.empty(N, dtype=torch.float64, device="cuda")
    draws = orc.uniforms(k0, k1, 0, N + 1)
    reports = {}
    for kind, fn, kw in (("dac", drs.dac_sampler, {}), ("dac_merge", drs.dac_sampler, {"mode": "merge"}),
                         ("ccf", drs.ccf_sampler, {})):
        out = fn(t, N, drs.RngStream(c["useed"]), uniforms_out=U, **kw)
        Ud = U.cpu().numpy()
        np.testing.assert_array_equal(Ud, Uo)  # K2 at 2^24 (repair path included when it fires)
        base = kind.split("_")[0]
        rep = parity.device_report(base, W, Ud, out, w, draws, W_ref=Wref)
        assert rep["exact_mismatches"] == 0, (kind, rep)
        assert rep["flips_unexplained"] == 0, (kind, rep)
        reports[kind] = rep
    out = drs.binary_sampler(t, N, drs.RngStream(c["useed"]))
    rep = parity.device_report("binary", W, None, out, w, draws[:N], W_ref=Wref)
    assert rep["exact_mismatches"] == 0 and rep["flips_unexplained"] == 0, rep
    # the spike block's run was drawn (k_merge_heavy path) and every index is in range
    assert out.min() >= 0 and out.max() < M
    print({k: (v["flips"], v["near_boundary_4ulp"], v["near_boundary_drift"]) for k, v in reports.items()})


def test_c5_deferred_equals_two_pass(drs, c5):
    """Config 5 at full size through both kinds of table: the single-pass
    (deferred, level 1 in-tile) table's W, formed on the device, is the
    two-pass table's W bit for bit over all 2^30 entries, and every sampler
    returns the same 2^24 indices from both (test_c5_full_size_bit_exact pins
    the deferred one against the oracle)."""
    w, c = c5
    N = c["N"]
    wd = torch.from_numpy(w).cuda()
    td = drs.build_weight_table(wd)
    tt = drs.build_weight_table(wd, deferred=False)
    del wd
    assert td.deferred and not tt.deferred
    assert torch.equal(td.device_cum, tt.device_values)
    for fn, kw in ((drs.dac_sampler, {}), (drs.dac_sampler, {"mode": "merge"}), (drs.ccf_sampler, {}),
                   (drs.binary_sampler, {})):
        a = fn(td, N, drs.RngStream(c["useed"]), device=True, **kw)
        b = fn(tt, N, drs.RngStream(c["useed"]), device=True, **kw)
        assert torch.equal(a, b), (fn.__name__, kw)


@pytest.mark.parametrize("cfg", ["c1", "c2", "c3"])
def test_boundary_report_device_mode(drs, cfg):
    """The north star's proximity report at c1-c3: device W and U vs the
    reference association; flips confined to the drift set; exact on the
    device's own W and U."""
    from bench import CONFIGS, make_weights
    from oracle import oracle as orc
    from oracle import parity

    c = CONFIGS[cfg]
    w = make_weights(cfg)
    t = drs.build_weight_table(w)
    N = c["N"]
    k0, k1 = orc.key_of(c["useed"])
    draws = orc.uniforms(k0, k1, 0, N + 1)
    Wref, _ = orc.port_build_table(w)
    U = torch.empty(N, dtype=torch.float64, device="cuda")
    for kind, fn in (("dac", drs.dac_sampler), ("ccf", drs.ccf_sampler)):
        out = fn(t, N, drs.RngStream(c["useed"]), uniforms_out=U)
        rep = parity.device_report(kind, t.cum, U.cpu().numpy(), out, w, draws, W_ref=Wref)
        assert rep["ok"], rep
    out = drs.binary_sampler(t, N, drs.RngStream(c["useed"]))
    rep = parity.device_report("binary", t.cum, None, out, w, draws[:N], W_ref=Wref)
    assert rep["ok"], rep


def test_exhaustive_tables_size8_digest(drs, golden):
    """Every table of size <= 8 over {0, 1, 2} (9,832 tables; reference
    tests/helpers.py:53-76): W built on the device, its boundary query set
    matched by every GPU matcher; the SHA-256 over (W, u, indices) equals the
    digest of the reference's own outputs (tests/golden, make_golden.py)."""
    import hashlib

    from tests.helpers import ReplayStream

    h = hashlib.sha256()
    count = 0
    for raw in enumerate_weight_tables(8):
        t = drs.build_weight_table(raw)
        W = t.cum
        u = boundary_query_set(W)
        e = drs.dac_match(u, t)
        for other in (drs.ccf_match(u, t), drs.dac_match(u, t, mode="merge"), drs.dac_match(u, t, mode="search"),
                      drs.binary_sampler(t, u.shape[0], ReplayStream(u))):
            np.testing.assert_array_equal(other, e)
        h.update(W.tobytes())
        h.update(u.tobytes())
        h.update(e.astype(np.int64).tobytes())
        count += 1
    assert count == int(golden["exh_count"])
    assert h.digest() == golden["exh_digest"].tobytes()


def test_c4_full_bank_bit_exact(drs, orc):
    """Config 4 at the bench's full size (B = 4096 filters of M_f = 16384,
    N_f = 256, SURVEY 8(d) field): W, U and indices of every filter
    bit-exact against the oracle twin of the batched kernel, which equals
    the per-filter build_weight_table + dac_sampler loop; and the reference
    association report over a prefix of the bank."""
    from bench import CONFIGS, make_weights, parity_block

    c = CONFIGS["c4"]
    w = make_weights("c4")
    B, Nf = w.shape[0], c["Nf"]
    assert B == 4096 and w.shape[1] == c["Mf"]
    streams = [drs.RngStream(c["useed"], (b,)) for b in range(B)]
    keys = np.array([[s.key[0], s.key[1], s.position] for s in streams], dtype=np.uint64)
    out, U, W = drs.resample_batched(w, Nf, streams, return_uniforms=True, return_tables=True)
    eo, Uo, Wo, st = orc.resample_batched(w, Nf, keys)
    assert st == 0
    np.testing.assert_array_equal(W, Wo)
    np.testing.assert_array_equal(U, Uo)
    np.testing.assert_array_equal(out, eo)
    rep = parity_block("c4", "dac", "auto", w)
    assert rep["ok"], rep


def test_sharded_nccl_two_gpus():
    """The W-sharded table and sampler over NCCL on two GPUs (runs only when
    two are visible): the gathered indices equal the single-GPU sampler's."""
    import os
    import subprocess
    import sys
    from pathlib import Path

    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    root = Path(__file__).resolve().parents[1]
    script = root / "tests" / "nccl_two_gpu.py"
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                        "--master-addr", "127.0.0.1", "--master-port", "29533", str(script)],
                       capture_output=True, text=True, timeout=600, cwd=str(root),
                       env={**os.environ, "PYTHONPATH": str(root)})
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "NCCL_TWO_GPU_OK" in r.stdout
