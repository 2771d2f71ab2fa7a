"""Either side of the resampling path on the GPU.

* ``gather_states``: the step after resampling -- particle states by index
  (an EnGMF state row is d = 40 fp64, weightgen.py:37).
* ``histogram``: ``np.bincount(indices, minlength=m)`` (bench.py:241).
* ``chi_square_statistic`` / ``verify_statistics``: the reference's Pearson
  goodness of fit (bench.py:221-246) with the counting and the statistic on
  the device; the draws come from the GPU samplers.

There is no CPU fallback: every step is a ``libdrs.so`` kernel.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._tensors import is_device_tensor, read_status, status_word, to_device_f64
from .cdf import WeightTable, build_weight_table
from .randkit import RngStream
from .samplers import binary_sampler, ccf_sampler, dac_sampler

__all__ = ["gather_states", "histogram", "chi_square_statistic", "GofReport", "verify_statistics",
           "dirichlet_uniform", "SAMPLER_ORDER"]

SAMPLER_ORDER = ("dac", "ccf", "binary")  # bench.py:41
_SAMPLERS = {"dac": dac_sampler, "ccf": ccf_sampler, "binary": binary_sampler}


def _to_device_i64(x) -> tuple[torch.Tensor, bool]:
    if is_device_tensor(x):
        return x.to(torch.int64).contiguous(), False
    a = np.ascontiguousarray(x, dtype=np.int64)
    return torch.from_numpy(a).to(_lib.device()), True


def gather_states(states, indices, *, divisor: int = 1):
    """Rows ``states[indices // divisor]`` (the resampled particles).

    ``states``: (K, d) float64 (numpy or CUDA tensor); ``indices``: int64[N]
    from a sampler.  ``divisor`` maps a mixture-component index to its
    particle (EnGMF: component = particle * N_Y + center, divisor = N_Y).
    Host inputs give a numpy (N, d) array, device inputs a CUDA tensor.
    """
    s, host = to_device_f64(states)
    if s.ndim == 1:
        s = s.reshape(-1, 1)
    if s.ndim != 2 or s.shape[0] == 0:
        raise ValueError("states must be (K, d) with K >= 1")
    idx, _ = _to_device_i64(indices)
    idx = idx.reshape(-1)
    K, d = int(s.shape[0]), int(s.shape[1])
    out = torch.empty((idx.numel(), d), dtype=torch.float64, device=s.device)
    st = status_word()
    _lib.check(_lib.lib().dr_gather_rows(s.data_ptr(), K, d, idx.data_ptr(), idx.numel(), int(divisor),
                                         out.data_ptr(), st.data_ptr(), _lib.stream_handle()), "dr_gather_rows")
    if read_status(st) & _lib.ST_OUT_OF_SUPPORT:
        raise IndexError("index out of range for the states array")
    return out.cpu().numpy() if host else out


def histogram(indices, m: int, *, device: bool = False):
    """``np.bincount(indices, minlength=m)`` computed on the device (int64)."""
    idx, host = _to_device_i64(indices)
    idx = idx.reshape(-1)
    counts = torch.empty(int(m), dtype=torch.int64, device=_lib.device())
    st = status_word()
    _lib.check(_lib.lib().dr_histogram(idx.data_ptr(), idx.numel(), int(m), counts.data_ptr(), st.data_ptr(),
                                       _lib.stream_handle()), "dr_histogram")
    if read_status(st) & _lib.ST_OUT_OF_SUPPORT:
        raise ValueError("index outside [0, m)")
    return counts if (device or not host) else counts.cpu().numpy()


def chi_square_statistic(counts, table: WeightTable, n_draws: int) -> float:
    """Pearson sum((observed - expected)^2 / expected) with expected =
    n_draws * table.weights() (bench.py:221-225, 241-242), on the device."""
    c, _ = _to_device_i64(counts)
    M = table.size
    if c.numel() != M:
        raise ValueError("need one count per table entry")
    L = _lib.lib()
    ws = torch.empty(int(L.dr_chi_square_workspace(M)) // 8, dtype=torch.float64, device=_lib.device())
    out = torch.empty(1, dtype=torch.float64, device=_lib.device())
    _lib.check(L.dr_chi_square(c.data_ptr(), table.device_cum.data_ptr(), M, int(n_draws), out.data_ptr(),
                               ws.data_ptr(), ws.numel() * 8, _lib.stream_handle()), "dr_chi_square")
    return float(out.item())


def dirichlet_uniform(m: int, stream: RngStream) -> np.ndarray:
    """m iid standard exponentials (weightgen.py:54-59), from the Philox stream."""
    m = int(m)
    if m < 1:
        raise ValueError("m must be >= 1")
    return -np.log(stream.uniforms(m))


@dataclass
class GofReport:
    """Chi-square goodness-of-fit result for one sampler (bench.py:91-100)."""

    sampler: str
    m: int
    n: int
    chi_square: float
    dof: int
    passed: bool


def verify_statistics(seed: int = 0, m: int = 16, n_draws: int = 1_000_000,
                      alpha: float = 1e-3) -> list[GofReport]:
    """bench.py:228-246 on the GPU: n_draws from a fixed m-component Dirichlet
    table per sampler (each its own substream), counted and scored on the
    device; pass = statistic below the upper-alpha chi-square quantile."""
    from scipy.stats import chi2

    root = RngStream(seed)
    table = build_weight_table(dirichlet_uniform(m, root.substream(0)))
    critical = float(chi2.isf(alpha, m - 1))
    reports = []
    for k, name in enumerate(SAMPLER_ORDER):
        idx = _SAMPLERS[name](table, n_draws, root.substream(1 + k), device=True)
        counts = histogram(idx, m, device=True)
        stat = chi_square_statistic(counts, table, n_draws)
        reports.append(GofReport(name, m, n_draws, stat, m - 1, stat < critical))
    return reports
