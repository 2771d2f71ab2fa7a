"""Where the end-to-end time of one public dac_sampler call goes (c3)."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
import paper_2604_01356_b200 as drs  # noqa: E402
from paper_2604_01356_b200 import _lib  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
c = bench.CONFIGS[cfg]
table = drs.build_weight_table(bench.make_weights(cfg))
N = c["N"]
st = drs.RngStream(c["useed"])
U = torch.empty(N, dtype=torch.float64, device="cuda")
out = torch.empty(N, dtype=torch.int64, device="cuda")


def clock(fn, k=200):
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(k):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / k * 1e6


def dev_sync():
    drs.dac_sampler(table, N, st, device=True, out=out, uniforms_out=U)
    torch.cuda.current_stream().synchronize()


print(f"{cfg}: device result + sync            {clock(dev_sync):8.1f} us")
print(f"{cfg}: device result, no sync (launch)  {clock(lambda: drs.dac_sampler(table, N, st, device=True, out=out, uniforms_out=U)):8.1f} us")
print(f"{cfg}: host result (public call)         {clock(lambda: drs.dac_sampler(table, N, st)):8.1f} us")
print(f"{cfg}: host result, U given              {clock(lambda: drs.dac_sampler(table, N, st, uniforms_out=U)):8.1f} us")
pin = torch.empty(N, dtype=torch.int64, pin_memory=True)
print(f"{cfg}: pinned alloc only                 {clock(lambda: torch.empty(N, dtype=torch.int64, pin_memory=True)):8.1f} us")
print(f"{cfg}: stream sync only                  {clock(lambda: torch.cuda.current_stream().synchronize()):8.1f} us")
print(f"{cfg}: stream_handle                     {clock(_lib.stream_handle, 2000):8.1f} us")
print(f"{cfg}: D2H copy of out into pinned       {clock(lambda: (pin.copy_(out, non_blocking=True), torch.cuda.current_stream().synchronize())):8.1f} us")
