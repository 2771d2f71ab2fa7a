"""Generate tests/golden/golden.npz by running the REFERENCE implementation.

Run in the build container (where /root/reference exists):

    NUMBA_CACHE_DIR=/tmp/nc PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Everything stored here is an output of /root/reference/pkg/src/dacresample
(build_weight_table, sorted_uniforms, ccf_match, dac_match, binary_sampler,
_repair_open_strict) on seeded inputs; the inputs themselves are either
stored or regenerable from the seeds recorded next to them.  The reference's
random draws come through a duck-typed stream serving numpy-Philox draws
(the generator this package uses), so the same draws can be replayed into
the device and oracle paths.  The GPU box never reads /root/reference; it
reads only this file.
"""

from __future__ import annotations

import hashlib
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, "/root/reference/pkg/tests")

import dacresample as ref  # noqa: E402
from dacresample import randkit as ref_randkit  # noqa: E402
from helpers import boundary_query_set, enumerate_weight_tables, linear_scan_bulk  # noqa: E402

OUT = Path(__file__).resolve().with_name("golden.npz")


class PhiloxStream:
    """RngStream duck type serving numpy Philox(SeedSequence(seed)) draws."""

    def __init__(self, seed, spawn_key=()):
        self._gen = np.random.Generator(np.random.Philox(np.random.SeedSequence(seed, spawn_key=spawn_key)))
        self.draws = 0

    def uniforms(self, k):
        self.draws += k
        return self._gen.random(int(k))


class ReplayStream:
    def __init__(self, values):
        self._v = np.asarray(values, dtype=np.float64)
        self.draws = 0

    def uniforms(self, k):
        out = self._v[self.draws:self.draws + k].copy()
        self.draws += k
        return out


def random_case(rng, max_m=4096, zero_frac=0.15):
    """test_acceptance.py:56-72 case generator (table + strictly increasing u)."""
    m = int(np.exp(rng.uniform(0.0, np.log(max_m)))) if max_m > 1 else 1
    n = int(np.exp(rng.uniform(0.0, np.log(m)))) if m > 1 else 1
    raw = rng.random(m)
    raw[rng.random(m) < zero_frac] = 0.0
    if raw.sum() == 0.0:
        raw[0] = 1.0
    table = ref.build_weight_table(raw)
    u = rng.random(n)
    boundaries = np.unique(table.cum[table.cum > 0.0])
    k = min(n // 3, boundaries.shape[0])
    if k:
        u[:k] = rng.choice(boundaries, size=k, replace=False)
    u = np.unique(u[u > 0.0])
    if u.shape[0] == 0:
        u = np.array([0.5])
    return raw, table, u


def main():
    g = {}

    # ---- 1. build_weight_table on assorted raw weights (exact reference W)
    rng = np.random.default_rng(20261019)
    raws = [np.array([2.0, 1.0, 1.0]), np.array([1.0]), np.array([1.0, 0.0, 0.0]), np.array([0.0, 1.0]),
            np.array([0.0, 0.3, 0.0, 0.7, 0.0])]
    for m in (2, 7, 33, 100, 1000, 8447, 8448, 8449, 20000):
        raws.append(rng.random(m))
    for m in (500, 9000):
        r = rng.random(m)
        r[rng.random(m) < 0.3] = 0.0
        raws.append(r)
    raws.append(np.exp(4.0 * rng.standard_normal(30000)))  # heavy tail (config 3 shape)
    raws.append(0.999 ** np.arange(5000.0))                # geometric (bench.py:44)
    raws.append(np.exp(np.random.default_rng(1001).standard_normal(2 ** 16)))  # config 1 weights
    for i, r in enumerate(raws):
        g[f"tbl_raw_{i}"] = r
        g[f"tbl_cum_{i}"] = ref.build_weight_table(r).cum.copy()
    g["tbl_count"] = np.array(len(raws))

    # ---- 2. matcher equivalence cases (acceptance criterion 1 generator, seed 0xACCE)
    rng = np.random.default_rng(0xACCE)
    Ws, Us, Es, mo, no = [], [], [], [0], [0]
    for _ in range(300):
        _, table, u = random_case(rng)
        e_ccf = ref.ccf_match(u, table)
        e_dac = ref.dac_match(u, table)
        e_bin = ref.binary_sampler(table, u.shape[0], ReplayStream(u))
        e_lin = linear_scan_bulk(table, u)
        assert np.array_equal(e_ccf, e_lin) and np.array_equal(e_dac, e_lin) and np.array_equal(e_bin, e_lin)
        Ws.append(table.cum)
        Us.append(u)
        Es.append(e_dac)
        mo.append(mo[-1] + table.size)
        no.append(no[-1] + u.shape[0])
    g["mc_W"] = np.concatenate(Ws)
    g["mc_U"] = np.concatenate(Us)
    g["mc_idx"] = np.concatenate(Es)
    g["mc_moff"] = np.array(mo)
    g["mc_noff"] = np.array(no)

    # ---- 3. exhaustive tables of size <= 8 over {0,1,2}: digest of reference outputs
    h = hashlib.sha256()
    count = 0
    for raw in enumerate_weight_tables(8, grid=(0.0, 1.0, 2.0)):
        table = ref.build_weight_table(raw)
        u = boundary_query_set(table)
        e = ref.dac_match(u, table)
        assert np.array_equal(e, ref.ccf_match(u, table))
        h.update(table.cum.tobytes())
        h.update(u.tobytes())
        h.update(e.astype(np.int64).tobytes())
        count += 1
    g["exh_digest"] = np.frombuffer(h.digest(), dtype=np.uint8)
    g["exh_count"] = np.array(count)

    # ---- 4. sorted_uniforms through the reference with Philox draws
    su_cases = [(2001, 1024), (7, 1), (8, 2), (9, 17), (10, 1000), (11, 5000), (12, 70000)]
    for i, (seed, n) in enumerate(su_cases):
        g[f"su_U_{i}"] = ref.sorted_uniforms(PhiloxStream(seed), n)
    g["su_cases"] = np.array(su_cases)

    # ---- 5. replayed draws, including the collapse / repair path
    rp_cases = [
        np.array([0.5, 0.5, 0.5]),                                   # test_randkit.py:47-51
        np.exp([-100.0, -1.0, -100.0]),                              # test_randkit.py:102-114
        np.array([0.5, 1 - 2.0 ** -53, 1 - 2.0 ** -53, 0.5]),        # two vanishing spacings
        np.array([1 - 2.0 ** -53, 1 - 2.0 ** -53, 1 - 2.0 ** -53, 1e-300]),  # collapse at 0
        np.array([1e-300, 1 - 2.0 ** -53, 1 - 2.0 ** -53]),          # collapse at 1
        np.concatenate([[0.3], np.full(40, 1 - 2.0 ** -53), [0.2], np.full(5, 1 - 2.0 ** -52), [0.7]]),
    ]
    for i, d in enumerate(rp_cases):
        n = d.shape[0] - 1
        g[f"rp_draws_{i}"] = d
        g[f"rp_U_{i}"] = ref.sorted_uniforms(ReplayStream(d), n)
    g["rp_count"] = np.array(len(rp_cases))
    v = np.array([0.1, 0.1, 0.1, 0.5, 0.5, 1.0, 1.0])
    g["repair_in"] = v
    vv = v.copy()
    ref_randkit._repair_open_strict(vv)
    g["repair_out"] = vv

    # ---- 6. config-1 sampler outputs (M = 2^16, N = 2^10) with Philox(2001) draws
    table = ref.build_weight_table(raws[-1])
    for name, fn in (("dac", ref.dac_sampler), ("ccf", ref.ccf_sampler)):
        g[f"c1_{name}"] = fn(table, 1024, PhiloxStream(2001))
    g["c1_binary"] = ref.binary_sampler(table, 1024, PhiloxStream(2001))

    np.savez_compressed(OUT, **g)
    print(f"wrote {OUT} ({OUT.stat().st_size / 1e6:.2f} MB), {count} exhaustive tables")


if __name__ == "__main__":
    main()
