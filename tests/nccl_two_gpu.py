"""Worker of tests/test_gpu_baseline_configs.py::test_sharded_nccl_two_gpus (one rank per GPU, NCCL).

Builds a W-sharded table over the ranks, samples with both communication
modes, gathers, and compares with the single-GPU dac_sampler on the whole
table (bit-exact: the sharded association's W differs from the single-GPU
table only by the shard split, so the comparison is against the oracle's
sharded table and sorted uniforms)."""

import os
import sys

import numpy as np
import torch
import torch.distributed as dist


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
    import paper_2604_01356_b200 as drs
    from oracle import oracle as orc

    M, N = (1 << 22) + 17, (1 << 18) + 5
    rng = np.random.default_rng(1005)
    w = np.exp(2 * rng.standard_normal(M))
    w[5000:6024] = (w.sum() - w[5000:6024].sum()) / 3 / 1024
    a, b = M * rank // world, M * (rank + 1) // world
    table = drs.build_sharded_table(torch.from_numpy(w[a:b]).cuda())
    Wo, To, _ = orc.build_table_sharded(w, world)
    np.testing.assert_array_equal(table.cum.cpu().numpy(), Wo[a:b])
    k0, k1 = orc.key_of(2005)
    Uo, _ = orc.sorted_uniforms(k0, k1, 0, N)
    expect = orc.match("dac", Wo, Uo)
    for comm in ("allgather", "none"):
        out, rng8 = drs.sharded_dac_sampler(table, N, drs.RngStream(2005), gather=True, comm=comm)
        np.testing.assert_array_equal(out.cpu().numpy(), expect)
    dist.barrier()
    if rank == 0:
        print("NCCL_TWO_GPU_OK")
    dist.destroy_process_group()


if __name__ == "__main__":
    sys.exit(main())
