"""The W-sharded table and sampler with the real device steps in two
processes (two ranks sharing cuda:0, collectives over gloo).

This is a functional check of the multi-process path -- DeviceShardOps,
the all-gathers, the windows, the capacity re-run, gather=True -- with no
kernel waiting on another rank (the collectives are host-side); the NCCL
version runs in test_gpu_baseline_configs.py::test_sharded_nccl_two_gpus when
two GPUs are visible.  The gathered indices must equal the oracle's DaC on
the oracle's sharded table and U.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _weights(M):
    rng = np.random.default_rng(1005)
    w = np.exp(2 * rng.standard_normal(M))
    w[rng.random(M) < 0.05] = 0.0
    off = int(rng.integers(0, M - 1024))
    w[off:off + 1024] = (w.sum() - w[off:off + 1024].sum()) / 3 / 1024
    return w


def _worker(rank, world, port, M, N, mode, q):
    import sys
    from pathlib import Path

    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        import paper_2604_01356_b200 as drs
        from paper_2604_01356_b200 import sharded

        w = _weights(M)
        if mode == "tinycap":
            sharded.slice_capacity = lambda table, n, tile, g=None: (8, 2)
        a, b = M * rank // world, M * (rank + 1) // world
        table = drs.build_sharded_table(torch.from_numpy(w[a:b]).cuda())
        outs = []
        for comm in ("allgather", "none"):
            out, rng = drs.sharded_dac_sampler(table, N, drs.RngStream(2005), gather=True, comm=comm)
            outs.append(out.cpu().numpy())
        q.put((rank, "ok", (table.cum.cpu().numpy(), outs)))
    except Exception as e:  # reported to the parent, which fails the test
        q.put((rank, "error", repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,M,N,mode", [(2, (1 << 20) + 5, (1 << 16) + 3, "ok"), (3, 200003, 70001, "ok"),
                                             (2, 300000, 20000, "tinycap")])
def test_sharded_ranks_on_one_gpu(orc, world, M, N, mode):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, M, N, mode, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
    assert all(r[1] == "ok" for r in res), res
    w = _weights(M)
    Wo, To, st = orc.build_table_sharded(w, world)
    np.testing.assert_array_equal(np.concatenate([r[2][0] for r in res]), Wo)
    k0, k1 = orc.key_of(2005)
    Uo, _ = orc.sorted_uniforms(k0, k1, 0, N)
    expect = orc.match("dac", Wo, Uo)
    for r in res:
        for out in r[2][1]:
            np.testing.assert_array_equal(out, expect)
