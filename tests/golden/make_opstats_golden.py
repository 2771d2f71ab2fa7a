"""Generate tests/golden/opstats.npz by running the REFERENCE's instrumented twins.

Run in the build container (where /root/reference exists):

    NUMBA_CACHE_DIR=/tmp/nc PYTHONPATH=/root/reference/pkg/src python tests/golden/make_opstats_golden.py

For every matcher case of golden.npz (the acceptance-1 generator, seed
0xACCE) and a few equal-weight / heavy-tailed tables of the verify_complexity
shape (bench.py:249-310), the OpStats of the reference's ccf_match
(samplers.py:178-188), dac_match (:213-232) and binary_sampler on the same
uniforms replayed (:249-252): rows of (comparisons, probes, max_depth).
The GPU box never reads /root/reference; it reads only this file.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")

import dacresample as ref  # noqa: E402

HERE = Path(__file__).resolve().parent


class ReplayStream:
    def __init__(self, values):
        self._v = np.asarray(values, dtype=np.float64)
        self.draws = 0

    def uniforms(self, k):
        out = self._v[self.draws:self.draws + k].copy()
        self.draws += k
        return out


def counts(table, u):
    rows = []
    for kind in ("ccf", "dac", "binary"):
        s = ref.OpStats()
        if kind == "ccf":
            ref.ccf_match(u, table, stats=s)
        elif kind == "dac":
            ref.dac_match(u, table, stats=s)
        else:
            ref.binary_sampler(table, u.shape[0], ReplayStream(u), stats=s)
        rows.append((s.comparisons, s.probes, s.max_depth))
    return rows


def main():
    g = dict(np.load(HERE / "golden.npz"))
    mo, no = g["mc_moff"], g["mc_noff"]
    out = []
    for i in range(len(mo) - 1):
        table = ref.WeightTable(g["mc_W"][mo[i]:mo[i + 1]])
        u = g["mc_U"][no[i]:no[i + 1]]
        out.append(counts(table, u))
    extra_W, extra_U, eo, en = [], [], [0], [0]
    ex = []
    rng = np.random.default_rng(0x0957)
    for n, ratio, kind in ((100, 1, "flat"), (100, 100, "flat"), (1000, 1, "flat"), (1000, 100, "flat"),
                           (3000, 50, "heavy"), (5000, 2, "zeros")):
        m = n * ratio
        if kind == "flat":
            w = np.full(m, 1.0 / m)
        elif kind == "heavy":
            w = np.exp(4.0 * rng.standard_normal(m))
        else:
            w = rng.random(m)
            w[rng.random(m) < 0.5] = 0.0
        table = ref.build_weight_table(w)
        u = np.sort(rng.random(n))
        u = np.unique(u[u > 0.0])
        ex.append(counts(table, u))
        extra_W.append(table.cum)
        extra_U.append(u)
        eo.append(eo[-1] + table.size)
        en.append(en[-1] + u.shape[0])
    np.savez_compressed(HERE / "opstats.npz", mc_counts=np.array(out, dtype=np.int64),
                        ex_counts=np.array(ex, dtype=np.int64), ex_W=np.concatenate(extra_W),
                        ex_U=np.concatenate(extra_U), ex_moff=np.array(eo), ex_noff=np.array(en))
    print("wrote", HERE / "opstats.npz", len(out), "cases +", len(ex))


if __name__ == "__main__":
    main()
