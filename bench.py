#!/usr/bin/env python
"""Benchmark of the resampling hot path (driver contract).

Default workload (BASELINE.json "metric", config 3): dac_sampler at
M = 2^26 heavy-tailed weights (log w ~ N(0, 4^2), seed 1003), N = 2^16 draws
(stream seed 2003).  A step is one sampler call: sorted uniforms + search,
with the table already built and resident (the reference's timed region,
bench.py:193-204).  Metric = algorithmic bytes (8M + 16N) / step time, plus
samples/s.  A step is one public-API call (device-resident result); L2 is
flushed (256 MiB write) before every timed step; steps are timed one by one
with CUDA events on the launching stream.  The same call replayed from a
CUDA graph (stream position on the device) is reported beside it.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c1..c5]
                  [--sampler dac|ccf|binary] [--mode auto|merge|search]
                  [--impl drs|reference]

--impl reference times the reference algorithm's CPU implementation (the
oracle's C port of the numba kernels + numpy pipeline, pinned bit-exact to
the reference) on this host's cores, same config and metric.
Under torchrun every rank runs an independent replica of the single-GPU
workload (weak scaling) except config c5, which shards one M = 2^30 table
over the ranks (one 24-byte-per-rank all-gather) and config c4, which
shards the 4096 filters by rank.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CONFIGS = {
    "c1": dict(M=1 << 16, N=1 << 10, sigma=1.0, wseed=1001, useed=2001),
    "c2": dict(M=1 << 20, N=1 << 20, sigma=1.0, wseed=1002, useed=2002),
    "c3": dict(M=1 << 26, N=1 << 16, sigma=4.0, wseed=1003, useed=2003),
    "c4": dict(B=4096, Mf=16384, Nf=256, wseed=1004, useed=2004),
    "c5": dict(M=1 << 30, N=1 << 24, sigma=2.0, wseed=1005, useed=2005),
}
METRIC = "weights-scanned GB/s (frac of HBM peak) + samples/sec, M=2^26 N=2^16"


def peak_hbm():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return float(json.loads(p.read_text())["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


# ------------------------------------------------------------------ inputs
def make_weights(cfg_name, rank=0, world=1):
    c = CONFIGS[cfg_name]
    if cfg_name == "c4":
        rng = np.random.default_rng(c["wseed"])
        B, Mf = c["B"], c["Mf"]
        lo, hi = B * rank // world, B * (rank + 1) // world
        pi = rng.dirichlet(np.ones(64), size=B)[lo:hi]
        out = np.empty((hi - lo, Mf))
        for b in range(hi - lo):  # chi-square field per filter, row-major (n, p)
            frng = np.random.default_rng([c["wseed"], lo + b])
            q = frng.chisquare(6, size=(256, 64))
            out[b] = np.exp(np.log(1 / 256) + np.log(pi[b])[None, :] - 0.5 * q).reshape(Mf)
        return out
    M = c["M"]
    if cfg_name == "c5":
        return make_c5_weights(rank, world)
    rng = np.random.default_rng(c["wseed"])
    return np.exp(c["sigma"] * rng.standard_normal(M))


C5_CHUNK = 1 << 24


def make_c5_weights(rank=0, world=1):
    """Config 5: w = exp(2 g), g ~ N(0, 1), drawn as 64 chunks of
    2^24 (chunk k from default_rng([1005, k]) -- per-chunk generators, so a rank
    can draw any chunk without drawing the ones before it), plus a block of
    1024 contiguous entries at a seeded offset (default_rng([1005, 999])) set
    to (total - block) / 3 / 1024, where total is the ACTUAL sum of the field
    (chunk sums np.sum, added in chunk order) and block the block's own sum:
    the block holds exactly 25% of the final mass.  Rank g of `world` gets
    its contiguous range [g M / world, (g + 1) M / world); every rank draws
    all chunks once to form the total (identical on every rank)."""
    c = CONFIGS["c5"]
    M = c["M"]
    a, b = M * rank // world, M * (rank + 1) // world
    off = int(np.random.default_rng([c["wseed"], 999]).integers(0, M - 1024))
    w = np.empty(b - a)
    total = 0.0
    block = 0.0
    for k in range(M // C5_CHUNK):
        g = np.exp(2.0 * np.random.default_rng([c["wseed"], k]).standard_normal(C5_CHUNK))
        total += float(g.sum())
        k0, k1 = k * C5_CHUNK, (k + 1) * C5_CHUNK
        blo, bhi = max(off, k0), min(off + 1024, k1)
        if blo < bhi:
            block += float(g[blo - k0:bhi - k0].sum())
        s0, s1 = max(a, k0), min(b, k1)
        if s0 < s1:
            w[s0 - a:s1 - a] = g[s0 - k0:s1 - k0]
    spike = (total - block) / 3.0 / 1024
    lo, hi = max(a, off), min(b, off + 1024)
    if lo < hi:
        w[lo - a:hi - a] = spike
    return w


# ------------------------------------------------------------------ clocks
class ClockSampler:
    def __init__(self, dev_index):
        self.dev = dev_index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        while not self._stop.is_set():
            try:
                r = subprocess.run(["nvidia-smi", "-i", str(self.dev), f"--query-gpu={q}", "--format=csv,noheader,nounits"],
                                   capture_output=True, text=True, timeout=5)
                if r.returncode == 0 and r.stdout.strip():
                    self.rows.append([x.strip() for x in r.stdout.strip().split(",")])
            except Exception:
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > i + 2 and r[i + 2] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def cdiv_(a, b):
    return -(-a // b)


# ---------------------------------------------------------------- drs arm
def run_drs(args, rank, world, local_rank, cfg=None, light=False):
    """One config on this rank; rank 0's JSON line.  ``light``: the timed
    steps, the dominant kernel and e2e only (the scaling blocks)."""
    import torch
    import torch.distributed as dist

    import paper_2604_01356_b200 as drs

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    cfg = cfg or args.config
    c = CONFIGS[cfg]
    alt = None
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def barrier():
        if world > 1:
            dist.barrier()

    flush_r = torch.zeros(256 << 20, dtype=torch.uint8, device=dev).view(torch.int32) if args.flush == "write+read" else None

    def l2_flush():
        # a 256 MiB write evicts everything but leaves L2 full of its own dirty lines, which the
        # timed kernel would then have to write back (~126 MB, ~19 us at the copy peak, charged to
        # whatever runs next); the read sweep of a second buffer replaces them by clean lines
        flush.fill_(1)
        if flush_r is not None:
            torch.sum(flush_r)

    # ---- untimed setup (the reference builds its table untimed too)
    if cfg == "c4":
        w_host = make_weights(cfg, rank, world)
        w = torch.from_numpy(w_host).to(dev)
        B, Mf, Nf = w.shape[0], c["Mf"], c["Nf"]
        mk = lambda: drs.BatchedStreams(  # noqa: E731
            [drs.RngStream(c["useed"], (rank * 100000 + b,)) for b in range(B)])
        bstreams, e2e_streams = mk(), mk()
        alg_bytes = B * (8 * Mf + 16 * Nf)
        samples = B * Nf

        def step():
            # stream positions live on the device and advance there
            return drs.resample_batched(w, Nf, bstreams, return_uniforms=True, check=False, device=True)

        launches_per_step = 2  # the bank's uniforms, then one cluster per filter
        kernel_step = step
        w_pinned = torch.from_numpy(w_host).pin_memory()
        # end to end: pinned host weights in, host indices out (status read included)
        e2e_step = lambda: drs.resample_batched(w_pinned, Nf, e2e_streams)  # noqa: E731
        e2e_h2d, e2e_d2h = 8 * B * Mf, 8 * B * Nf + 4
    elif cfg == "c5" and world > 1:
        w_host = make_weights(cfg, rank, world)
        table = drs.build_sharded_table(torch.from_numpy(w_host).to(dev), deferred=args.table == "deferred")
        N = c["N"]
        stream = drs.RngStream(c["useed"])
        alg_bytes = (8 * c["M"]) // world + 16 * N // world
        samples = N // world
        comm = args.comm

        def step():
            # status not read in the timed loop (no host round trip); the
            # windows hold mean + 12 sd of the slice
            return drs.sharded_dac_sampler(table, N, stream, comm=comm, check=False)

        other = "none" if comm == "allgather" else "allgather"
        alt = (other, lambda: drs.sharded_dac_sampler(table, N, stream, comm=other, check=False))
        # tile totals (1/G of them, or all for comm none), [all-gather], stage, chain,
        # tile range, regenerate, finish, match
        launches_per_step = 7
        kernel_step = step
        e2e_stream = drs.RngStream(c["useed"], (1,))
        slices = []

        def e2e_step():
            # the public call, then this rank's slice of indices to the host
            out, rng = drs.sharded_dac_sampler(table, N, e2e_stream, comm=comm)
            i0, i1 = rng[:2].tolist()
            slices.append(i1 - i0)
            return out[: i1 - i0].cpu()

        e2e_h2d, e2e_d2h = 0, 8 * (N // world)
    else:
        w_host = make_weights(cfg)
        table = drs.build_weight_table(w_host, deferred=args.table == "deferred")
        M, N = c["M"], c["N"]
        stream = drs.RngStream(c["useed"], (rank,))
        alg_bytes = 8 * M + 16 * N
        samples = N
        sampler = {"dac": drs.dac_sampler, "ccf": drs.ccf_sampler, "binary": drs.binary_sampler}[args.sampler]
        kw = {"mode": args.mode} if args.sampler == "dac" else {}
        out_buf = torch.empty(N, dtype=torch.int64, device=dev)
        if args.sampler != "binary":
            kw["uniforms_out"] = torch.empty(N, dtype=torch.float64, device=dev)

        def eager_step():
            return sampler(table, N, stream, device=True, out=out_buf, **kw)

        step = eager_step
        graph_step = None
        fused = args.sampler == "dac" and args.mode != "merge" and M > 16 * N and (N + 1) <= 148 * 512
        # sorted uniforms = pass 1 + chain + pass 2 + finalize, then the search
        # (merge: k_merge_tiles, plus k_merge_heavy for the long runs when N > 4096)
        merge_launches = 5 + (1 if N > 4096 else 0)
        dac_merge = args.mode == "merge" or (args.mode == "auto" and M <= 16 * N)
        launches_per_step = {"binary": 1, "ccf": merge_launches}.get(
            args.sampler, 1 if fused else (merge_launches if dac_merge else 5))
        if args.graph and not light:
            # the same call captured once in a CUDA graph; the stream position
            # lives on the device, so every replay draws fresh uniforms
            dstream = drs.DeviceRngStream(c["useed"], (rank,))
            side = torch.cuda.Stream(device=dev)
            side.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(side):
                sampler(table, N, dstream, device=True, out=out_buf, **kw)
                graph = torch.cuda.CUDAGraph()
                with torch.cuda.graph(graph, stream=side):
                    sampler(table, N, dstream, device=True, out=out_buf, **kw)
            torch.cuda.current_stream().wait_stream(side)

            def graph_step():
                graph.replay()
        # the dominant kernel alone: the search over a fixed U
        U = drs.randkit.sorted_uniforms_device(drs.RngStream(c["useed"], (rank, 7)), N)
        match = {"dac": lambda: drs.dac_match(U, table, check=False, mode=args.mode),
                 "ccf": lambda: drs.ccf_match(U, table, check=False),
                 "binary": lambda: drs.samplers._lower_bounds(table, U)}[args.sampler]
        # the dominant kernel: the fused sampler kernel when the step is that one
        # launch, else the search over a fixed U
        kernel_step = eager_step if (fused and args.sampler == "dac") else match
        # the reference's call, dac_sampler(table, n, stream) (its timed region,
        # bench.py:193-204): host result, no uniforms output
        e2e_kw = {"mode": args.mode} if args.sampler == "dac" else {}
        e2e_step = lambda: sampler(table, N, stream, **e2e_kw)  # noqa: E731
        e2e_h2d, e2e_d2h = 0, 8 * N

    # ---- warm-up
    for _ in range(args.warmup):
        step()
        kernel_step()
    torch.cuda.synchronize()
    s = torch.cuda.current_stream()

    def timed(fn, k):
        starts = [torch.cuda.Event(enable_timing=True) for _ in range(k)]
        ends = [torch.cuda.Event(enable_timing=True) for _ in range(k)]
        for i in range(k):
            l2_flush()
            starts[i].record(s)
            fn()
            ends[i].record(s)
        torch.cuda.synchronize()
        return [a.elapsed_time(b) for a, b in zip(starts, ends)]

    # ---- timed region: per-step events, L2 flushed before each step
    barrier()
    torch.cuda.synchronize()
    with ClockSampler(local_rank) as clk:
        time.sleep(0.2)  # the first nvidia-smi sample is taken before the timed steps start
        step()
        torch.cuda.synchronize()
        step_ms = timed(step, args.steps)
    barrier()
    alt_ms = None
    if alt is not None:  # the other communication mode of the sharded sampler, same discipline
        for _ in range(3):
            alt[1]()
        barrier()
        torch.cuda.synchronize()
        a_ms = float(sum(timed(alt[1], args.steps)))
        if world > 1:
            t = torch.tensor([a_ms], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            a_ms = float(t.item())
        alt_ms = a_ms / args.steps
    graph_ms = None
    if not light and cfg not in ("c4",) and not (cfg == "c5" and world > 1) and locals().get("graph_step") is not None:
        for _ in range(3):
            graph_step()
        graph_ms = statistics.median(timed(graph_step, args.steps))
    total_ms = float(sum(step_ms))
    if world > 1:
        t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps

    # ---- dominant kernel alone (live, same flush discipline)
    k_ms = []
    for _ in range(args.steps):
        l2_flush()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        kernel_step()
        b.record(s)
        torch.cuda.synchronize()
        k_ms.append(a.elapsed_time(b))
    kernel_ms = statistics.median(k_ms)

    # ---- K1 on its own: build_weight_table from device-resident raw weights
    # (16 M algorithmic bytes -- read w, write W)
    table_build = None
    if not light and cfg == "c5" and world > 1:
        # the sharded table's build (the public collective call: local scan,
        # the 24-byte-per-rank all-gather, finalize), both kinds of shard;
        # max over ranks
        w_dev = torch.from_numpy(w_host).to(dev)
        sb = {}
        for kind in ("deferred", "two-pass"):
            drs.build_sharded_table(w_dev, deferred=kind == "deferred")
            ms = []
            for _ in range(max(3, min(args.steps, 10))):
                l2_flush()
                barrier()
                torch.cuda.synchronize()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(s)
                drs.build_sharded_table(w_dev, deferred=kind == "deferred")
                b.record(s)
                torch.cuda.synchronize()
                ms.append(a.elapsed_time(b))
            t = torch.tensor([statistics.median(ms)], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            sb[kind] = float(t.item())
        del w_dev
        Mg = w_host.size
        table_build = {"ms": sb["deferred"], "two_pass_ms": sb["two-pass"], "per_rank_entries": Mg,
                       "GB/s_per_rank": 16 * Mg / (sb["deferred"] * 1e-3) / 1e9,
                       "frac": 16 * Mg / (sb["deferred"] * 1e-3) / 1e9 / peak_hbm()[0],
                       "timed": "build_sharded_table (public call incl. the all-gather of the shard totals), "
                                "max over ranks, CUDA events, L2 flushed",
                       "note": "deferred shards: dr_shard_scan_deferred + all-gather + dr_shard_finalize_deferred "
                               "(16 B/entry, no pass after the collective); two_pass: dr_shard_scan + "
                               "dr_shard_finalize (48 B/entry); the sampled table is --table"}
    if not light and (cfg in ("c1", "c2", "c3") or (cfg == "c5" and world == 1)):
        w_dev = torch.from_numpy(w_host).to(dev)
        from paper_2604_01356_b200 import _lib as dlib

        Lb = dlib.lib()
        M_ = c["M"]
        Wb = torch.empty(M_, dtype=torch.float64, device=dev)
        ib = torch.empty(int(Lb.dr_index_entries(M_)), dtype=torch.float64, device=dev)
        stb = torch.zeros(1, dtype=torch.int32, device=dev)
        wsb_ptr, wsb_n = dlib.workspace(Lb.dr_workspace_bytes(dlib.OP_TABLE, M_, 0, 0))

        def time_build(fn, reps=max(3, min(args.steps, 10))):
            fn()
            ms = []
            for _ in range(reps):
                l2_flush()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(s)
                fn()
                b.record(s)
                torch.cuda.synchronize()
                ms.append(a.elapsed_time(b))
            return statistics.median(ms)

        def abi_build(name):  # the C ABI on preallocated buffers: the kernels alone
            return lambda: dlib.check(getattr(Lb, name)(w_dev.data_ptr(), M_, Wb.data_ptr(), ib.data_ptr(),
                                                        stb.data_ptr(), wsb_ptr, wsb_n, dlib.stream_handle()), name)

        tbm = time_build(abi_build("dr_build_table_deferred"))
        tb2 = time_build(abi_build("dr_build_table"))
        tb_api = time_build(lambda: drs.build_weight_table(w_dev, check=False))
        del w_dev, Wb, ib
        table_build = {"ms": tbm, "GB/s": 16 * M_ / (tbm * 1e-3) / 1e9,
                       "frac": 16 * M_ / (tbm * 1e-3) / 1e9 / peak_hbm()[0],
                       "algorithmic_bytes": 16 * M_, "launches": 3 if 32 < cdiv_(M_, 8448) <= 16384 else 4,
                       "note": "single pass (dr_build_table_deferred): read w once, write the table once "
                               "(+ level 1 of the index, M/16); then the tile chain + the levels above 1 in one "
                               "launch (k_table_tail; the chain and levels kernels for > 16384 tiles), then the guide",
                       "two_pass_ms": tb2,
                       "two_pass_note": "dr_build_table: pass 1 reads w, pass 2 reads w again and writes W",
                       "timed": "the C ABI on preallocated table buffers (CUDA events, L2 flushed)",
                       "api_ms": tb_api,
                       "api_note": "build_weight_table(w_dev): the public call, allocating the table"}
        tk = ROOT / "profiles" / f"traffic_k1_{cfg}.json"
        if tk.exists():  # the single pass's DRAM bytes from a committed ncu capture
            kt = json.loads(tk.read_text())
            table_build["single_pass_kernel"] = {"traffic": kt.get("bytes_per_launch"),
                                                 "duration_us_ncu": kt.get("duration_us_ncu"),
                                                 "source": kt.get("source")}

    # ---- the particle filter's resampling step (the paper's loop: new weights every
    # step): build_weight_table + the benchmarked sampler, device-resident weights in
    # and indices out, events; and end to end from pinned host weights to host indices
    filter_step = None
    if not light and cfg in ("c1", "c2", "c3"):
        w_dev = torch.from_numpy(w_host).to(dev)
        w_pin = torch.from_numpy(w_host).pin_memory()
        fs_stream = drs.RngStream(c["useed"], (rank, 11))

        def fstep_dev():
            t_ = drs.build_weight_table(w_dev, check=False)
            return sampler(t_, N, fs_stream, device=True, out=out_buf, **kw)

        def fstep_e2e():
            t_ = drs.build_weight_table(w_pin)  # pinned host weights: H2D inside, status read
            return sampler(t_, N, fs_stream, **kw)  # host indices

        for _ in range(2):
            fstep_dev()
            fstep_e2e()
        torch.cuda.synchronize()
        fs_ms = []
        for _ in range(max(3, min(args.steps, 10))):
            l2_flush()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            fstep_dev()
            b.record(s)
            torch.cuda.synchronize()
            fs_ms.append(a.elapsed_time(b))
        reps = max(3, min(args.steps, 10))
        t0 = time.perf_counter()
        for _ in range(reps):
            fstep_e2e()
        torch.cuda.synchronize()
        fe = (time.perf_counter() - t0) / reps
        fsm = statistics.median(fs_ms)
        fb = 16 * c["M"] + 16 * N  # table (read w, write W) + sampler (U + indices); W read by the search is extra
        filter_step = {"ms": fsm, "samples_per_s": N / (fsm * 1e-3), "algorithmic_bytes": fb,
                       "GB/s": fb / (fsm * 1e-3) / 1e9,
                       "timed": "build_weight_table (device weights) + one sampler call, CUDA events, L2 flushed",
                       "e2e": {"ms_per_step": 1e3 * fe, "h2d_bytes_per_step": 8 * c["M"], "d2h_bytes_per_step": 8 * N,
                               "timer": "host perf_counter: pinned host weights -> table -> sampler -> host indices"}}
        del w_dev, w_pin

    # ---- the step after resampling: the resampled particle states,
    # EnGMF layout (component = particle * N_Y + center, N_Y = M / N, d = 40):
    # sampler + gather kernel (two calls) against resample_and_gather (the rows
    # copied from the indices in registers in the single-kernel regime)
    resample_gather = None
    if not light and cfg in ("c1", "c2", "c3") and args.sampler == "dac":
        ny, dd = c["M"] // N, 40
        xs = torch.randn((N, dd), dtype=torch.float64, device=dev)
        rg_stream = drs.RngStream(c["useed"], (rank, 12))

        def rg_two():
            i_ = drs.dac_sampler(table, N, rg_stream, device=True, out=out_buf)
            return drs.gather_states(xs, i_, divisor=ny, check=False)  # no status read: no host sync

        def rg_fused():
            return drs.resample_and_gather(table, N, rg_stream, xs, divisor=ny)

        def ev_median(fn, reps):
            for _ in range(3):
                fn()
            ts = []
            for _ in range(reps):
                l2_flush()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(s)
                fn()
                b.record(s)
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b))
            return statistics.median(ts)

        reps = max(5, min(args.steps, 20))
        t_two, t_fused = ev_median(rg_two, reps), ev_median(rg_fused, reps)
        i_f, r_f = drs.resample_and_gather(table, N, drs.RngStream(c["useed"], (rank, 13)), xs, divisor=ny)
        i_r = drs.dac_sampler(table, N, drs.RngStream(c["useed"], (rank, 13)), device=True)
        same = bool(torch.equal(i_f, i_r) and torch.equal(r_f, xs[torch.div(i_r, ny, rounding_mode="floor")]))
        rb = 2 * 8 * dd * N  # row reads + row writes
        resample_gather = {"rows": N, "d": dd, "divisor": ny, "row_bytes": rb,
                           "ms_sampler_then_gather": t_two, "ms_fused": t_fused,
                           "speedup": t_two / t_fused, "identical": same,
                           "timed": "CUDA events, L2 flushed, device table/states/result"}
        del xs

    # ---- the north star's recast beside the headline (c3 dac auto searches the index and touches
    # ~9.5 MB; mode="merge" streams all of W through shared-memory tiles, so its algorithmic bytes are
    # its physical bytes and its fraction is a roofline fraction): same call, same flush discipline
    merge_recast = None
    if not light and cfg == "c3" and args.sampler == "dac" and args.mode != "merge":
        mr_stream = drs.RngStream(c["useed"], (rank, 14))
        mr_step = lambda: drs.dac_sampler(table, N, mr_stream, device=True, out=out_buf, mode="merge")  # noqa: E731
        for _ in range(3):
            mr_step()
        mr_ms = statistics.median(timed(mr_step, max(5, min(args.steps, 20))))
        tm = ROOT / "profiles" / f"traffic_{cfg}_dac_merge.json"
        mr_traffic = json.loads(tm.read_text()) if tm.exists() else {}
        merge_recast = {"mode": "merge", "ms_per_step": mr_ms, "GB/s": alg_bytes / (mr_ms * 1e-3) / 1e9,
                        "frac": alg_bytes / (mr_ms * 1e-3) / 1e9 / peak_hbm()[0],
                        "kernel_ncu": mr_traffic or None,
                        "timed": "one dac_sampler(mode='merge') call per step (uniforms + k_merge_tiles + the "
                                 "long-run helper), CUDA events, L2 flushed"}

    # ---- end to end through the public API, host result (and host weights for c4)
    e2e = None
    if e2e_step is not None:
        # every call returns a host result (it synchronises), so calls are timed
        # back to back; at least ~0.2 s of calls after 10 warm-ups, so a single
        # host hiccup does not dominate a 40 us call
        for _ in range(10):
            e2e_step()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e2e_step()
        torch.cuda.synchronize()
        one = time.perf_counter() - t0
        # the same count on every rank: the sharded call holds a collective
        e2e_calls = max(args.steps, min(2000, int(0.2 / max(one, 1e-6)))) if world == 1 else args.steps
        t0 = time.perf_counter()
        for _ in range(e2e_calls):
            e2e_step()
        torch.cuda.synchronize()
        e2e_s = (time.perf_counter() - t0) / e2e_calls
        if world > 1:  # the slowest rank
            t = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_s = float(t.item())
        e2e = {"value": world * alg_bytes / e2e_s / 1e9, "unit": "GB/s", "samples_per_s": world * samples / e2e_s,
               "ms_per_step": 1e3 * e2e_s, "h2d_bytes_per_step": e2e_h2d, "d2h_bytes_per_step": e2e_d2h,
               "timer": "host perf_counter around the public call (result copied to host)", "calls": e2e_calls}

    value = world * alg_bytes / (ms_per_step * 1e-3) / 1e9
    peak, peak_src = peak_hbm()
    achieved = alg_bytes / (kernel_ms * 1e-3) / 1e9
    traffic = None
    tp = ROOT / "profiles" / f"traffic_{cfg}_{args.sampler}_{args.mode}.json"
    if tp.exists():
        traffic = json.loads(tp.read_text()).get("bytes_per_launch")
        if world > 1 and cfg in ("c4", "c5"):
            traffic = None  # captured on one GPU for the whole bank / table: not this rank's launch
    line = {
        "metric": METRIC if cfg == "c3" else f"weights-scanned GB/s + samples/sec, {cfg}",
        "value": value,
        "unit": "GB/s",
        "samples_per_s": world * samples / (ms_per_step * 1e-3),
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_per_step,
        "higher_is_better": True,
        "scaling": "strong" if (cfg == "c5" and world > 1) else "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (seeded numpy weights, SURVEY.md 8(d)); Philox draws",
        "config": {
            "workload": cfg, **{k: v for k, v in c.items()}, "sampler": args.sampler, "mode": args.mode,
            "table": "per-filter tables formed in shared memory (never stored)" if cfg == "c4" else args.table,
            "timed": ("per step: every filter's table scan + sorted uniforms + search, raw weights resident "
                      "(the reference's per-filter loop, cdf.py:59-89 + samplers.py:262-266)") if cfg == "c4"
            else "sorted uniforms + search per step, table resident (reference bench.py:193-204)",
            "l2": ("flushed (256 MiB write, then a 256 MiB read sweep of a second buffer so that no dirty "
                   "flush lines are written back inside the timed region) before every timed step; steps timed "
                   "individually") if args.flush == "write+read"
            else "flushed (256 MiB write) before every timed step; steps timed individually",
            "parallelism": ("shard-W" if cfg == "c5" else ("shard-filters" if cfg == "c4" else "replicas")) + f"x{world}",
        },
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "kernel_ms": kernel_ms, "peak_source": peak_src,
                     "algorithmic_bytes_per_launch": alg_bytes,
                     "physical_frac": (traffic / (kernel_ms * 1e-3) / 1e9 / peak) if traffic else None},
        "e2e": e2e,
        "gpu_launches": launches_per_step * args.steps,
        "table_build": table_build,
        "filter_step": filter_step,
        "resample_gather": resample_gather,
        "merge_recast": merge_recast,
        "clocks": clk.summary(),
        "step_ms_min": min(step_ms), "step_ms_median": statistics.median(step_ms),
        "timing": "one public-API sampler call per step (device result), CUDA events on the launching stream",
        "steps_ms": [round(x, 5) for x in step_ms],
        "graph_replay_ms_per_step_median": graph_ms,
    }
    if alt is not None:
        line["config"]["comm"] = args.comm
        line["alt_comm"] = {"comm": alt[0], "ms_per_step": alt_ms,
                            "value": world * alg_bytes / (alt_ms * 1e-3) / 1e9}
    if world == 1 and args.parity and not light:
        line["parity"] = parity_block(cfg, args.sampler, args.mode, w_host, locals().get("table"))
    return line, (alg_bytes, samples)


# ---------------------------------------------------------- parity checker
def parity_block(cfg, sampler, mode, w_host, table=None):
    """The north star's device-mode correctness counters for one call of the
    benchmarked sampler on this config (oracle/parity.py; the CHECKER, run
    after the timed region at N = 1 on rank 0, never timed): exact-mode
    mismatches of the reference matcher on the device's own W and U, W / U
    ulp histograms against the reference association, u within 4 ulp and
    within the measured drift of a boundary, index flips, unexplained flips."""
    import time as _t

    import torch

    import paper_2604_01356_b200 as drs
    from oracle import oracle as orc
    from oracle import parity

    t0 = _t.perf_counter()
    c = CONFIGS[cfg]
    if cfg == "c4":
        # a bounded prefix of the bank: device W, U and indices against the
        # oracle twin bit for bit, and against the reference association
        Bs = 256
        w = w_host[:Bs]
        Mf, Nf = c["Mf"], c["Nf"]
        streams = [drs.RngStream(c["useed"], (b,)) for b in range(Bs)]
        keys = np.array([[s.key[0], s.key[1], s.position] for s in streams], dtype=np.uint64)
        out, U, W = drs.resample_batched(w, Nf, streams, return_uniforms=True, return_tables=True)
        eo, Uo, Wo, _ = orc.resample_batched(w, Nf, keys)
        agg = {"filters": Bs, "twin_mismatches": int(np.count_nonzero(out != eo) + np.count_nonzero(U != Uo)
                                                    + np.count_nonzero(W != Wo))}
        keys_sum = ("exact_mismatches", "near_boundary_4ulp", "near_boundary_drift", "flips", "flips_unexplained")
        for k in keys_sum:
            agg[k] = 0
        agg["W_max_ulp"] = agg["U_max_ulp"] = 0
        for b in range(Bs):
            draws = orc.uniforms(int(keys[b, 0]), int(keys[b, 1]), 0, Nf + 1)
            r = parity.device_report("dac", W[b], U[b], out[b], w[b], draws)
            for k in keys_sum:
                agg[k] += r[k]
            agg["W_max_ulp"] = max(agg["W_max_ulp"], r["W_max_ulp"])
            agg["U_max_ulp"] = max(agg["U_max_ulp"], r["U_max_ulp"])
        agg["ok"] = agg["twin_mismatches"] == 0 and agg["exact_mismatches"] == 0 and agg["flips_unexplained"] == 0
        agg["seconds"] = _t.perf_counter() - t0
        return agg
    N = c["N"]
    k0, k1 = orc.key_of(c["useed"])
    fn = {"dac": drs.dac_sampler, "ccf": drs.ccf_sampler, "binary": drs.binary_sampler}[sampler]
    kw = {"mode": mode} if sampler == "dac" else {}
    if sampler == "binary":
        out = fn(table, N, drs.RngStream(c["useed"]))
        draws, Ud = orc.uniforms(k0, k1, 0, N), None
    else:
        U = torch.empty(N, dtype=torch.float64, device="cuda")
        out = fn(table, N, drs.RngStream(c["useed"]), uniforms_out=U, **kw)
        draws, Ud = orc.uniforms(k0, k1, 0, N + 1), U.cpu().numpy()
        Uo, _ = orc.sorted_uniforms(k0, k1, 0, N)
    W = table.cum
    Wo, _ = orc.build_table(w_host)
    twin = int(np.count_nonzero(W != Wo)) + (int(np.count_nonzero(Ud != Uo)) if Ud is not None else 0)
    del Wo
    rep = parity.device_report(sampler, W, Ud, out, w_host, draws)
    rep["twin_mismatches"] = twin  # device W / U vs the oracle's device-association twins
    rep["ok"] = rep["ok"] and twin == 0
    rep["seconds"] = _t.perf_counter() - t0
    return rep


# ------------------------------------------------------------ CPU baseline
def cpu_baseline(cfg, sampler, seconds=10.0, threads=1):
    from oracle import oracle as orc

    c = CONFIGS[cfg]
    if cfg == "c4":
        # the reference's per-filter loop (build_weight_table + dac_sampler),
        # on a bounded prefix of the filter bank, scaled to the full bank
        w = make_weights(cfg)
        B, Mf, Nf = w.shape[0], c["Mf"], c["Nf"]
        k0, k1 = orc.key_of(c["useed"])
        Bs = max(threads, 64)
        el = orc.port_batched_throughput(w[:Bs], Nf, threads, 1, k0, k1)
        reps = 1
        Bs = int(min(B, max(Bs, Bs * seconds / max(el, 1e-6) / 2)))
        el = orc.port_batched_throughput(w[:Bs], Nf, threads, reps, k0, k1)
        per_step = el * B / Bs
        return {"value": B * (8 * Mf + 16 * Nf) / per_step / 1e9, "unit": "GB/s", "cores": threads, "kind": "port",
                "samples_per_s": B * Nf / per_step,
                "sample": f"c4 per-filter build_weight_table+dac_sampler loop over {Bs} of {B} filters "
                          f"({threads} thread(s)), {el:.1f} s, scaled to the bank; oracle C port of the reference",
                "ms_per_call": 1e3 * per_step}
    proxy = ""
    if cfg == "c5":
        cfg, proxy = "c3", " (c3-shaped proxy: the M=2^30 table needs ~27 GB host RAM and ~30 s to build)"
        c = CONFIGS[cfg]
    w = make_weights(cfg)
    W, _ = orc.port_build_table(w)
    M, N = c["M"], c["N"]
    k0, k1 = orc.key_of(c["useed"])
    one = orc.port_throughput(sampler, W, N, 1, 1, k0, k1)  # includes first-touch
    one = orc.port_throughput(sampler, W, N, 1, 1, k0, k1)
    calls = max(1, int(seconds / max(one, 1e-6) / threads))
    el = orc.port_throughput(sampler, W, N, threads, calls, k0, k1)
    per = el / calls  # wall time per call per thread (threads run concurrently)
    value = threads * (8 * M + 16 * N) / per / 1e9
    return {"value": value, "unit": "GB/s", "cores": threads, "kind": "port",
            "samples_per_s": threads * N / per,
            "sample": f"{cfg} {sampler}_sampler x{calls * threads} calls ({threads} thread(s)), {el:.1f} s, "
                      "oracle C port of the reference path (pinned bit-exact to the reference)" + proxy,
            "ms_per_call": 1e3 * per}


def reference_numba_baseline(cfg, seconds=3.0):
    """The reference package itself (numba, single-threaded: SPEC.md:359) on this
    host, when it is installed in baseline/_ref (pip install --no-deps --target
    baseline/_ref of /root/reference/pkg): each sampler timed the reference's
    way (bench.py:193-204: table built untimed, one call per timing, PCG64
    streams) for about `seconds`; the C port in cpu_baseline is the pinned
    restatement of the same code."""
    ref_dir = ROOT / "baseline" / "_ref"
    if cfg not in ("c1", "c2", "c3") or not (ref_dir / "dacresample").is_dir():
        return {"unavailable": "config without a single table, or baseline/_ref not installed"}
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/drs_numba_cache")
    sys.path.insert(0, str(ref_dir))
    try:
        import dacresample as ref
        from dacresample.samplers import warm_kernels
    except Exception as e:  # numba missing or the package broken: report, do not fail the bench
        return {"unavailable": f"import failed: {e!r}"[:200]}
    finally:
        sys.path.remove(str(ref_dir))
    c = CONFIGS[cfg]
    table = ref.build_weight_table(make_weights(cfg))
    warm_kernels()
    out = {"kind": "reference", "cores": 1, "package": "baseline/_ref/dacresample (numba)"}
    for name in ("dac", "ccf", "binary"):
        fn = getattr(ref, f"{name}_sampler")
        fn(table, c["N"], ref.RngStream(1))  # the read-only table specialisation compiles here
        st = ref.RngStream(c["useed"])
        calls, t0 = 0, time.perf_counter()
        while time.perf_counter() - t0 < seconds:
            fn(table, c["N"], st)
            calls += 1
        per = (time.perf_counter() - t0) / calls
        out[name] = {"ms_per_call": 1e3 * per, "value": (8 * c["M"] + 16 * c["N"]) / per / 1e9, "unit": "GB/s",
                     "samples_per_s": c["N"] / per, "calls": calls}
    return out


def host_info():
    """CPU model and core counts of this host (the CPU baselines' hardware)."""
    model = None
    try:
        for ln in Path("/proc/cpuinfo").read_text().splitlines():
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    try:
        usable = len(os.sched_getaffinity(0))
    except AttributeError:
        usable = os.cpu_count()
    return {"model": model, "os_cpu_count": os.cpu_count(), "usable_cpus": usable}


def run_reference(args):
    threads = os.cpu_count() or 1
    cb = cpu_baseline(args.config, args.sampler, seconds=max(5.0, min(30.0, 2.0 * args.steps)), threads=threads)
    line = {
        "impl": "reference",
        "metric": METRIC if args.config == "c3" else f"weights-scanned GB/s + samples/sec, {args.config}",
        "value": cb["value"], "unit": "GB/s", "samples_per_s": cb["samples_per_s"],
        "n_gpus": int(os.environ.get("WORLD_SIZE", "1")), "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": cb["ms_per_call"], "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded numpy weights); Philox draws",
        "config": {"workload": args.config, **CONFIGS[args.config], "sampler": args.sampler},
        "cpu_baseline": cb,
        "cpu_host": host_info(),
        "e2e": {"value": cb["value"], "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    return line


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--sampler", default="dac", choices=["dac", "ccf", "binary"])
    ap.add_argument("--mode", default="auto", choices=["auto", "merge", "search"])
    ap.add_argument("--impl", default="drs", choices=["drs", "reference"])
    ap.add_argument("--table", default="two-pass", choices=["deferred", "two-pass"],
                    help="the sampled (resident) table: two-pass W (built once, sampled many times: the "
                         "reference's timed region) or the single-pass deferred table (build_weight_table's "
                         "default; the table_build and filter_step lines, where it is rebuilt every step)")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--comm", default="allgather", choices=["allgather", "none"],
                    help="c5 sharded sampling: all-gather of spacing-tile totals, or none (every rank computes all)")
    ap.add_argument("--no-scaling-blocks", dest="scaling_blocks", action="store_false",
                    help="skip the c5 (W-sharded, strong) and c4 (filter-sharded, weak) blocks after the c3 headline")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: functional check of the multi-rank flow only (never a perf number)")
    ap.add_argument("--no-parity", dest="parity", action="store_false",
                    help="skip the device-mode parity block (oracle checker, after the timed region)")
    ap.add_argument("--flush", default="write", choices=["write", "write+read"],
                    help="L2 flush before every timed step: a 256 MiB write, or that write followed by a "
                         "256 MiB read sweep (no dirty flush lines left for the timed kernel to write back)")
    ap.add_argument("--no-graph", dest="graph", action="store_false",
                    help="time eager API calls instead of CUDA-graph replays")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # `bench.py --gpus N` launched directly: re-exec under torchrun, one rank per GPU
        import socket

        sk = socket.socket()
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
        sk.close()
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")  # stdout carries the one JSON line only
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), str(Path(__file__).resolve()),
               *sys.argv[1:]]
        os.execv(sys.executable, cmd)

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus and rank == 0:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; measuring {world} rank(s)", file=sys.stderr)

    if args.impl == "reference":
        if rank == 0:
            print(json.dumps(run_reference(args)), flush=True)
        return

    import torch
    import torch.distributed as dist

    if world > 1:
        if args.dist_backend == "nccl" and torch.cuda.device_count() < world:
            if rank == 0:
                print(json.dumps({"error": f"{world} ranks need {world} GPUs, {torch.cuda.device_count()} visible"}),
                      flush=True)
            sys.exit(1)
        torch.cuda.set_device(local_rank % torch.cuda.device_count())
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            dist.init_process_group("gloo")
        local_rank = local_rank % torch.cuda.device_count()
    line, _ = run_drs(args, rank, world, local_rank)
    if args.scaling_blocks and args.config == "c3":
        # the multi-GPU configs in the same run: c5 shards one M = 2^30 table over the
        # ranks (strong scaling; one GPU: the plain single-GPU sampler), c4 shards the
        # 4096 filters (weak in filters per rank: no collective)
        blocks = {}
        for cfg2 in ("c5", "c4"):
            import gc

            gc.collect()
            torch.cuda.empty_cache()
            b, _ = run_drs(args, rank, world, local_rank, cfg=cfg2, light=True)
            keep = ("value", "unit", "samples_per_s", "ms_per_step", "n_gpus", "scaling", "config", "roofline",
                    "e2e", "alt_comm", "gpu_launches", "step_ms_median")
            blocks[cfg2] = {k: b[k] for k in keep if k in b}
        line["scaling_blocks"] = blocks
    if rank == 0:
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(args.config, args.sampler, seconds=args.cpu_seconds)
            # the reference's other CPU paths on the same workload (north star: "next to the
            # reference's CPU divide-and-conquer and Carpenter paths ... with the core count stated")
            others = [] if args.config == "c4" else [s for s in ("dac", "ccf", "binary") if s != args.sampler]
            line["cpu_baselines"] = {args.sampler: line["cpu_baseline"],
                                     **{s: cpu_baseline(args.config, s, seconds=args.cpu_seconds / 2)
                                        for s in others}}
            line["cpu_host"] = host_info()
            line["cpu_baselines"]["reference_numba"] = reference_numba_baseline(args.config)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
