"""CPU: the oracle's single-pass (deferred) table restates dr_build_table's W.

``oracle.build_table_deferred`` splits the chained association of
drs_ref_chain_scan at the tile prefix (V = R + (Q + s), pairs {C_g, D_t});
its W = fl((C_g + (D_t + V)) / T) must equal the two-pass twin's W bit for
bit, and its index the direct index of that W.
"""

import numpy as np
import pytest


@pytest.mark.parametrize("M", [1, 2, 16, 17, 8447, 8448, 8449, 32 * 8448 + 3, 200_003, 262_144, 262_145, 600_001])
def test_deferred_twin_equals_two_pass_twin(orc, M):
    rng = np.random.default_rng(M)
    w = np.exp(3.0 * rng.standard_normal(M))
    w[rng.random(M) < 0.2] = 0.0
    if w.sum() == 0:
        w[0] = 1.0
    V, idx, W, st = orc.build_table_deferred(w)
    W2, st2 = orc.build_table(w)
    assert st == st2 == 0
    np.testing.assert_array_equal(W, W2)
    ns = orc.search_entries(M)
    ref_idx, l1 = orc.index_l1_local(V, orc.build_index(W2))
    np.testing.assert_array_equal(idx[:ns], ref_idx[:ns])
    T = idx[ns]
    assert idx[ns + 1] == (5.0 if l1 else 1.0) and T > 0
    assert l1 == (M > 16 * 16384)  # level 1 in-tile once the top guide sits above it
    P = idx[ns + 4:].reshape(-1, 2)
    assert P.shape[0] == -(-M // 8448) and P[0, 0] == 0.0 and P[0, 1] == 0.0
    t = np.arange(M) // 8448
    S = P[t, 0] + (P[t, 1] + V)
    Wf = np.minimum(S / T, 1.0)
    Wf[-1] = 1.0
    np.testing.assert_array_equal(Wf, W)
    assert S[-1] == T  # the pinned top is T / T


def test_deferred_twin_status(orc):
    assert orc.build_table_deferred(np.array([0.0, 0.0]))[3] & 0x2
    assert orc.build_table_deferred(np.array([-1.0, 1.0]))[3] & 0x1
    assert orc.build_table_deferred(np.array([1e308, 1e308]))[3] & 0x4
