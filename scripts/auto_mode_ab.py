"""dac_sampler merge vs search step time (events, L2 flushed) around the auto threshold M <= 16 N."""
import statistics
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2604_01356_b200 as drs  # noqa: E402

flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
rng = np.random.default_rng(1)
for lm in (20, 22, 24, 26):
    M = 1 << lm
    t = drs.build_weight_table(torch.from_numpy(np.exp(2 * rng.standard_normal(M))).cuda(), deferred=False)
    for ratio in (1, 2, 4, 8, 16, 32, 64):
        N = M // ratio
        out = torch.empty(N, dtype=torch.int64, device="cuda")
        U = torch.empty(N, dtype=torch.float64, device="cuda")
        res = {}
        for mode in ("merge", "search"):
            st = drs.RngStream(3)
            ms = []
            for r in range(12):
                flush.fill_(r)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                drs.dac_sampler(t, N, st, device=True, out=out, uniforms_out=U, mode=mode)
                b.record()
                torch.cuda.synchronize()
                ms.append(a.elapsed_time(b))
            res[mode] = 1e3 * statistics.median(ms[3:])
        print(f"M=2^{lm} M/N={ratio:3d}: merge {res['merge']:8.1f} us  search {res['search']:8.1f} us  -> {'merge' if res['merge'] < res['search'] else 'search'}", flush=True)
