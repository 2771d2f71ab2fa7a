import statistics, sys
import numpy as np, torch
sys.path.insert(0, "/root/repo")
import paper_2604_01356_b200 as drs
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
rng = np.random.default_rng(1)
for lm in (26, 22):
    M = 1 << lm
    t = drs.build_weight_table(torch.from_numpy(np.exp(4 * rng.standard_normal(M))).cuda(), deferred=False)
    for N in (1 << 16, 75775, 75776, 1 << 17, 1 << 18, 303103, 303104, 1 << 19):
        for kind, kw in (("dac", {}), ("ccf", {})):
            fn = drs.dac_sampler if kind == "dac" else drs.ccf_sampler
            out = torch.empty(N, dtype=torch.int64, device="cuda"); U = torch.empty(N, dtype=torch.float64, device="cuda")
            st = drs.RngStream(3); ms = []
            for r in range(14):
                flush.fill_(r); a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(); fn(t, N, st, device=True, out=out, uniforms_out=U); b.record(); torch.cuda.synchronize(); ms.append(a.elapsed_time(b))
            print(f"M=2^{lm} N={N} {kind}: {1e3*statistics.median(ms[3:]):.1f} us", flush=True)
