"""ccf_sampler step time (events, L2 flushed) for u's-per-tile ratios around the merge-path threshold."""
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
for lm, ln in [tuple(int(x) for x in a.split(':')) for a in sys.argv[1:]] or ((24, 17), (24, 18), (24, 19), (24, 20), (26, 20), (26, 21), (22, 17), (22, 16)):
    M, N = 1 << lm, 1 << ln
    t = drs.build_weight_table(torch.from_numpy(np.exp(2 * rng.standard_normal(M))).cuda(), deferred=False)
    st = drs.RngStream(3)
    out = torch.empty(N, dtype=torch.int64, device="cuda")
    ms = []
    for r in range(15):
        flush.fill_(r)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        drs.ccf_sampler(t, N, st, device=True, out=out)
        b.record()
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    print(f"M=2^{lm} N=2^{ln} u/4096-tile={N * 4096 / M:7.1f}: {1e3 * statistics.median(ms[3:]):8.1f} us", flush=True)
