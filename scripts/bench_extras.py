"""Measurements of the SURVEY 8(f) rows (one JSON line).

* log-weight table (fused max -> exp -> scan) vs the unfused device pipeline
  (torch max + exp, then build_weight_table), M = 2^26 (c3's size);
* gather of resampled particle states (d = 40 fp64, the EnGMF state size);
* histogram + chi-square of the c3 draws.
CUDA-event timing, L2 flushed before each rep, median of reps.
"""
import json
import statistics
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2604_01356_b200 as drs  # noqa: E402
from bench import peak_hbm  # noqa: E402

flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def timeit(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    ts = []
    for r in range(reps):
        flush.fill_(r)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


peak = peak_hbm()[0]
res = {"metric": "SURVEY 8(f) rows", "unit": "ms / GB/s", "peak_hbm_gbs": peak}
M = 1 << 26
rng = np.random.default_rng(1003)
lw = torch.from_numpy(4.0 * rng.standard_normal(M)).cuda()
t_fused = timeit(lambda: drs.build_weight_table_from_log(lw, check=False))
t_unfused = timeit(lambda: drs.build_weight_table(torch.exp(lw - lw.max()), check=False))
t_plain = timeit(lambda: drs.build_weight_table(lw, check=False))
res["log_table"] = {"M": M, "fused_ms": t_fused, "unfused_ms": t_unfused, "plain_table_ms": t_plain,
                    "fused_alg_GBps": 16 * M / (t_fused * 1e-3) / 1e9,
                    "note": "fused: max reduction, pass 1 forms w = exp(lw - max) in SMEM (stored once), chain, pass 2; unfused: torch max/exp + build_weight_table"}
table = drs.build_weight_table(lw.exp().clamp_max(1e300), check=False)
for N in (1 << 16, 1 << 20):
    d = 40
    idx = drs.dac_sampler(table, N, drs.RngStream(2003), device=True)
    states = torch.from_numpy(rng.standard_normal((N, d))).cuda()
    sidx = (idx % N).contiguous()
    tg = timeit(lambda: drs.gather_states(states, sidx))
    res[f"gather_N{N}"] = {"N": N, "d": d, "ms": tg, "GBps": (2 * N * d * 8 + 8 * N) / (tg * 1e-3) / 1e9}
idx = drs.dac_sampler(table, 1 << 16, drs.RngStream(2003), device=True)
th = timeit(lambda: drs.histogram(idx, M, device=True))
counts = drs.histogram(idx, M, device=True)
tc = timeit(lambda: drs.chi_square_statistic(counts, table, 1 << 16))
res["histogram_c3"] = {"M": M, "N": 1 << 16, "ms": th, "note": "includes zeroing 8M bytes of counts"}
res["chi_square_c3"] = {"M": M, "ms": tc, "GBps": 16 * M / (tc * 1e-3) / 1e9}
print(json.dumps(res))
