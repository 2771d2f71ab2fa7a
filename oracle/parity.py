"""Device-mode parity report (north star) -- TEST INFRASTRUCTURE ONLY.

The checker behind the ``parity`` block of bench.py and the ``-m gpu`` parity
tests.  Given what the device produced for one sampler call (its W, its U, its
indices) and the raw weights / raw draws the call consumed, it reports:

1. *exact mode*: the reference's own matcher (the oracle port of
   ``_dac_kernel`` / ``_ccf_kernel`` / ``_binary_kernel``, samplers.py:93-146)
   run on the DEVICE's W and U must reproduce the device indices bit for bit
   (``exact_mismatches`` must be 0);
2. *reference association*: W_ref = the port of ``build_weight_table``
   (pairwise total, sequential cumsum: cdf.py:77-88) and U_ref = the port of
   ``sorted_uniforms`` on ``-np.log`` of the same draws (randkit.py:84-101):
   ulp histograms of W - W_ref and U - U_ref, the max absolute drifts, the
   number of u within 4 ulp of a boundary W_{j-1} / W_j (the north star's
   proximity rule), the number within the measured drift, and the index flips
   against the reference's indices.  Every flip must lie in the drift set: all
   boundaries between the device's and the reference's answer lie within
   drift_W + drift_U of u (``flips_unexplained`` must be 0).

Nothing here is imported by the product package; bench.py calls it after the
timed region, at N = 1 on rank 0 only (the checker, not the thing measured).
"""

from __future__ import annotations

import numpy as np

from . import oracle as orc

ULP_BINS = (0, 1, 2, 4, 16, 256, 4096, 65536)


def ulp_distance(a, b) -> np.ndarray:
    """|a - b| in units in the last place, for finite non-negative doubles."""
    ia = np.ascontiguousarray(a, dtype=np.float64).view(np.int64)
    ib = np.ascontiguousarray(b, dtype=np.float64).view(np.int64)
    return np.abs(ia - ib)


def ulp_histogram(d: np.ndarray) -> dict:
    """Counts of ulp distances in the bins 0, 1, 2, 3-4, 5-16, ..., > 65536."""
    out = {}
    lo = -1
    for hi in ULP_BINS:
        key = str(hi) if hi - lo == 1 else f"{lo + 1}-{hi}"
        out[key] = int(np.count_nonzero((d > lo) & (d <= hi)))
        lo = hi
    out[f">{ULP_BINS[-1]}"] = int(np.count_nonzero(d > ULP_BINS[-1]))
    return out


def _near_boundaries(W, u, j, tol_abs=None, tol_ulp=None):
    """Boolean per u: u lies within tol of W[j] or of W[j-1] (j = its index)."""
    hi = W[j]
    lo = np.where(j > 0, W[np.maximum(j - 1, 0)], 0.0)
    if tol_ulp is not None:
        near = ulp_distance(u, hi) <= tol_ulp
        near |= (j > 0) & (ulp_distance(u, lo) <= tol_ulp)
    else:
        near = np.abs(hi - u) <= tol_abs
        near |= (j > 0) & (np.abs(u - lo) <= tol_abs)
    return near


def device_report(kind: str, W_dev, U_dev, out_dev, raw_weights, draws, *, W_ref=None) -> dict:
    """The parity block for one device call.

    kind: "dac" | "ccf" | "binary".  ``draws``: the raw uniforms the call
    consumed (n + 1 for the sorted samplers, n for binary, in draw order);
    ``U_dev``: the device's sorted uniforms (None for binary, whose u are
    the draws themselves).  ``W_ref`` may be passed when already computed.
    """
    W_dev = np.ascontiguousarray(W_dev, dtype=np.float64)
    out_dev = np.ascontiguousarray(out_dev, dtype=np.int64)
    n = out_dev.shape[0]
    if kind == "binary":
        u_dev = np.ascontiguousarray(draws, dtype=np.float64)[:n]
        u_ref = u_dev
    else:
        u_dev = np.ascontiguousarray(U_dev, dtype=np.float64)
        u_ref, _ = orc.sorted_from_z(-np.log(np.asarray(draws, dtype=np.float64)), n, association="port")
    # 1. exact mode: the reference matcher on the device's own W and U
    exact = orc.match(kind, W_dev, u_dev)
    exact_mismatches = int(np.count_nonzero(exact != out_dev))
    # 2. against the reference association
    if W_ref is None:
        W_ref, _ = orc.port_build_table(raw_weights)
    e_ref = orc.match(kind, W_ref, u_ref)
    dW = ulp_distance(W_dev, W_ref)
    drift_W = float(np.max(np.abs(W_dev - W_ref))) if W_dev.size else 0.0
    if kind == "binary":
        dU = np.zeros(0, dtype=np.int64)
        drift_U = 0.0
    else:
        dU = ulp_distance(u_dev, u_ref)
        drift_U = float(np.max(np.abs(u_dev - u_ref))) if n else 0.0
    tol = drift_W + drift_U
    near4 = _near_boundaries(W_ref, u_ref, e_ref, tol_ulp=4)
    near_drift = _near_boundaries(W_ref, u_ref, e_ref, tol_abs=tol)
    flips = np.nonzero(out_dev != e_ref)[0]
    if flips.size:
        a = np.minimum(out_dev[flips], e_ref[flips])
        b = np.maximum(out_dev[flips], e_ref[flips])
        uf = u_ref[flips]
        # every boundary crossed between the two answers (W[a] .. W[b-1]) lies within the drift of u
        explained = (np.abs(W_ref[a] - uf) <= tol) & (np.abs(W_ref[b - 1] - uf) <= tol)
        unexplained = int(np.count_nonzero(~explained))
    else:
        unexplained = 0
    return {
        "kind": kind,
        "n": int(n),
        "m": int(W_dev.size),
        "exact_mismatches": exact_mismatches,
        "W_ulp_hist": ulp_histogram(dW),
        "U_ulp_hist": ulp_histogram(dU) if dU.size else None,
        "W_max_ulp": int(dW.max()) if dW.size else 0,
        "U_max_ulp": int(dU.max()) if dU.size else 0,
        "drift_W": drift_W,
        "drift_U": drift_U,
        "near_boundary_4ulp": int(np.count_nonzero(near4)),
        "near_boundary_drift": int(np.count_nonzero(near_drift)),
        "flips": int(flips.size),
        "flips_in_4ulp_set": int(np.count_nonzero(near4[flips])) if flips.size else 0,
        "flips_unexplained": unexplained,
        "ok": exact_mismatches == 0 and unexplained == 0,
    }
