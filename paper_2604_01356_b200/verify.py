"""Either side of the resampling path on the GPU.

* ``gather_states``: the step after resampling -- particle states by index
  (an EnGMF state row is d = 40 fp64, weightgen.py:37).
* ``resample_and_gather``: ``dac_sampler`` and that gather in one library
  call (``dr_sample_dac_gather``): in the single-kernel regime the rows are
  copied from the indices still in registers.
* ``histogram``: ``np.bincount(indices, minlength=m)`` (bench.py:241).
* ``chi_square_statistic`` / ``verify_statistics``: the reference's Pearson
  goodness of fit (bench.py:221-246) with the counting and the statistic on
  the device; the draws come from the GPU samplers.
* ``verify_complexity``: the reference's operation budgets (bench.py:249-310)
  on the OpStats the GPU samplers report (``dr_op_counts``: the reference's
  instrumented counts, computed exactly from the device's result).

There is no CPU fallback: every step is a ``libdrs.so`` kernel.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from ._tensors import is_device_tensor, read_status, status_word, to_device_f64
from .cdf import WeightTable, build_weight_table
from .randkit import DeviceRngStream, RngStream
from .samplers import OpStats, binary_sampler, ccf_sampler, dac_sampler
from . import samplers as _samplers

__all__ = ["gather_states", "resample_and_gather", "histogram", "chi_square_statistic", "GofReport", "verify_statistics",
           "ComplexityCell", "verify_complexity", "dirichlet_uniform", "SAMPLER_ORDER"]

SAMPLER_ORDER = ("dac", "ccf", "binary")  # bench.py:41
_SAMPLERS = {"dac": dac_sampler, "ccf": ccf_sampler, "binary": binary_sampler}


def _to_device_i64(x) -> tuple[torch.Tensor, bool]:
    if is_device_tensor(x):
        return x.to(torch.int64).contiguous(), False
    a = np.ascontiguousarray(x, dtype=np.int64)
    return torch.from_numpy(a).to(_lib.device()), True


def gather_states(states, indices, *, divisor: int = 1, check: bool = True):
    """Rows ``states[indices // divisor]`` (the resampled particles).

    ``states``: (K, d) float64 (numpy or CUDA tensor); ``indices``: int64[N]
    from a sampler.  ``divisor`` maps a mixture-component index to its
    particle (EnGMF: component = particle * N_Y + center, divisor = N_Y).
    Host inputs give a numpy (N, d) array, device inputs a CUDA tensor.
    ``check=False`` skips the status read (no host synchronisation; rows of
    out-of-range indices are then left unwritten).
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
    if check and read_status(st) & _lib.ST_OUT_OF_SUPPORT:
        raise IndexError("index out of range for the states array")
    return out.cpu().numpy() if host else out


def resample_and_gather(table: WeightTable, n: int, stream, states, *, divisor: int = 1, mode: str = "auto",
                        device: bool = False):
    """``idx = dac_sampler(table, n, stream)`` and ``gather_states(states, idx,
    divisor=divisor)`` as one call; same draws, same indices, same rows.

    ``stream``: RngStream or DeviceRngStream.  ``states``: (K, d) float64
    with ``(table.size - 1) // divisor < K``.  Returns ``(indices, rows)``:
    numpy for host states unless ``device``, else CUDA tensors.
    """
    if mode not in _lib.DAC_MODES:
        raise ValueError(f"unknown mode {mode!r}")
    if not isinstance(stream, (RngStream, DeviceRngStream)):
        raise TypeError("resample_and_gather needs an RngStream or DeviceRngStream")
    n, divisor = int(n), int(divisor)
    if n < 0:
        raise ValueError("n must be >= 0")
    if divisor < 1:
        raise ValueError("divisor must be >= 1")
    s_, host = to_device_f64(states)
    if s_.ndim == 1:
        s_ = s_.reshape(-1, 1)
    if s_.ndim != 2 or s_.shape[0] == 0:
        raise ValueError("states must be (K, d) with K >= 1")
    s_ = s_.contiguous()
    K, d = int(s_.shape[0]), int(s_.shape[1])
    if (table.size - 1) // divisor >= K:
        raise IndexError("index out of range for the states array")
    dev = _lib.device()
    idx = torch.empty(n, dtype=torch.int64, device=dev)
    rows = torch.empty((n, d), dtype=torch.float64, device=dev)
    if n:
        L = _lib.lib()
        sh = _lib.stream_handle()
        U = _samplers._scratch_uniforms(n, sh)
        st = _samplers._status_buf(sh)
        ws, wsb = _lib.workspace(_lib.workspace_bytes(_lib.OP_SORTED, n), sh)
        k0, k1, off, offd = _samplers._stream_args(stream, n + 1)
        _lib.check(L.dr_sample_dac_gather(table.device_values.data_ptr(), _samplers._ptr(table.device_index),
                                          table.size, k0, k1, off, offd, n, U.data_ptr(), idx.data_ptr(),
                                          s_.data_ptr(), K, d, divisor, rows.data_ptr(), st.data_ptr(),
                                          _lib.DAC_MODES[mode], ws, wsb, sh), "dr_sample_dac_gather")
    if host and not device:
        return idx.cpu().numpy(), rows.cpu().numpy()
    return idx, rows


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


@dataclass
class ComplexityCell:
    """Instrumented operation counts for one (N, ratio) cell vs their budgets (bench.py:103-124)."""

    n: int
    ratio: int
    m: int
    trials: int
    ccf_max_comparisons: int
    ccf_budget: int
    binary_max_probes: int
    dac_max_probes: int
    probe_budget: int
    dac_max_depth: int
    depth_budget: int
    dac_mean_probes: float
    dac_mean_budget: float
    violations: list[str] = field(default_factory=list)

    @property
    def ok(self) -> bool:
        return not self.violations


def verify_complexity(seed: int = 0, ns: tuple[int, ...] = (100, 1000), ratios: tuple[int, ...] = (1, 100, 1000),
                      trials: int = 50) -> list[ComplexityCell]:
    """bench.py:249-310 on the GPU samplers: equal-weight tables, per-sampler
    substreams, the hard budgets per run (CCF comparisons <= N + M - 1;
    binary and DaC probes <= N (ceil(log2 M) + 1); scope nesting <=
    ceil(log2 N) + 1) and the statistical one per cell (mean DaC probes <=
    4N (1 + log2(M/N + 1))), on the counts ``stats=`` reports."""
    root = RngStream(seed)
    cells = []
    cell_key = 0
    for n in ns:
        for ratio in ratios:
            cell_key += 1
            m = n * ratio
            table = build_weight_table(np.full(m, 1.0 / m))
            streams = {name: root.substream(cell_key).substream(k) for k, name in enumerate(SAMPLER_ORDER)}
            probe_budget = n * (math.ceil(math.log2(m)) + 1) if m > 1 else n
            ccf_budget = n + m - 1
            depth_budget = math.ceil(math.log2(n)) + 1 if n > 1 else 1
            dac_mean_budget = 4.0 * n * (1.0 + math.log2(m / n + 1.0))
            ccf_max = bin_max = dac_max = depth_max = 0
            dac_probes = []
            violations = []
            for _ in range(trials):
                s = OpStats()
                ccf_sampler(table, n, streams["ccf"], stats=s, device=True)
                ccf_max = max(ccf_max, s.comparisons)
                if s.comparisons > ccf_budget:
                    violations.append(f"ccf comparisons {s.comparisons} > {ccf_budget}")
                s = OpStats()
                binary_sampler(table, n, streams["binary"], stats=s, device=True)
                bin_max = max(bin_max, s.probes)
                if s.probes > probe_budget:
                    violations.append(f"binary probes {s.probes} > {probe_budget}")
                s = OpStats()
                dac_sampler(table, n, streams["dac"], stats=s, device=True)
                dac_max = max(dac_max, s.probes)
                depth_max = max(depth_max, s.max_depth)
                dac_probes.append(s.probes)
                if s.probes > probe_budget:
                    violations.append(f"dac probes {s.probes} > {probe_budget}")
                if s.max_depth > depth_budget:
                    violations.append(f"dac depth {s.max_depth} > {depth_budget}")
            dac_mean = float(np.mean(dac_probes))
            if dac_mean > dac_mean_budget:
                violations.append(f"dac mean probes {dac_mean:.1f} > {dac_mean_budget:.1f}")
            cells.append(ComplexityCell(
                n=n, ratio=ratio, m=m, trials=trials,
                ccf_max_comparisons=ccf_max, ccf_budget=ccf_budget,
                binary_max_probes=bin_max, dac_max_probes=dac_max,
                probe_budget=probe_budget, dac_max_depth=depth_max,
                depth_budget=depth_budget, dac_mean_probes=dac_mean,
                dac_mean_budget=dac_mean_budget, violations=violations,
            ))
    return cells
