"""The device-mode parity checker (oracle/parity.py) on CPU.

The device association's W and U are reproduced bit for bit by the oracle's
``drs_ref_*`` twins, so the report can be exercised here with those twins
standing in for the device outputs: zero exact-mode mismatches, every flip
against the reference association explained by the measured drift, and a
deliberately wrong index caught.
"""

import numpy as np

from oracle import parity


def _case(orc, M, N, sigma, seed):
    w = np.exp(sigma * np.random.default_rng(seed).standard_normal(M))
    W, _ = orc.build_table(w)
    k0, k1 = orc.key_of(seed + 1)
    draws = orc.uniforms(k0, k1, 0, N + 1)
    U, _ = orc.sorted_uniforms(k0, k1, 0, N)
    return w, W, U, draws


def test_report_on_device_twins(orc):
    for M, N, sigma in ((1 << 16, 1 << 10, 1.0), (1 << 20, 1 << 14, 4.0), (1 << 18, 1 << 18, 1.0)):
        w, W, U, draws = _case(orc, M, N, sigma, M + N)
        for kind in ("dac", "ccf"):
            out = orc.match(kind, W, U)
            rep = parity.device_report(kind, W, U, out, w, draws)
            assert rep["ok"] and rep["exact_mismatches"] == 0, rep
            assert rep["n"] == N and rep["m"] == M
            assert sum(rep["W_ulp_hist"].values()) == M
            assert sum(rep["U_ulp_hist"].values()) == N
            assert rep["near_boundary_4ulp"] <= rep["near_boundary_drift"] or rep["drift_W"] + rep["drift_U"] == 0
        out = orc.match("binary", W, draws[:N])
        rep = parity.device_report("binary", W, None, out, w, draws[:N])
        assert rep["ok"], rep


def test_report_catches_a_wrong_index(orc):
    w, W, U, draws = _case(orc, 4096, 512, 1.0, 3)
    out = orc.match("dac", W, U)
    out[100] += 7
    rep = parity.device_report("dac", W, U, out, w, draws)
    assert rep["exact_mismatches"] == 1 and rep["flips_unexplained"] >= 1 and not rep["ok"]


def test_ulp_histogram_bins():
    d = np.array([0, 0, 1, 2, 3, 4, 5, 16, 17, 70000])
    h = parity.ulp_histogram(d)
    assert h["0"] == 2 and h["1"] == 1 and h["2"] == 1 and h["3-4"] == 2 and h["5-16"] == 2
    assert h["17-256"] == 1 and h[">65536"] == 1
    assert sum(h.values()) == d.size
