"""Host-side cost of one dac_sampler call at c3, split into ctypes, launch,
kernel and the host-result path (prints one line per item, microseconds)."""
import sys, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_2604_01356_b200 as drs
from paper_2604_01356_b200 import _lib, samplers
from paper_2604_01356_b200._tensors import host_result_i64
import bench

table = drs.build_weight_table(bench.make_weights("c3"))
N = bench.CONFIGS["c3"]["N"]
L = _lib.lib()
s = _lib.stream_handle()


def clock(name, fn, k=1000):
    for _ in range(20):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(k):
        fn()
    dt = (time.perf_counter() - t0) / k * 1e6
    torch.cuda.synchronize()
    print(f"{name:48s} {dt:7.2f} us", flush=True)


W = table.device_cum
U = samplers._scratch_uniforms(N, s)
o = torch.empty(N, dtype=torch.int64, device="cuda")
ho = host_result_i64(N)
sb = samplers._status_buf(s)
ws, wsb = _lib.workspace(_lib.workspace_bytes(_lib.OP_SORTED, N), s)
idx = table.device_index
bad = (W.data_ptr(), idx.data_ptr(), 0, 1, 2, 0, 0, N, U.data_ptr(), o.data_ptr(), sb.data_ptr(), 0, ws, wsb, s)
dev = (W.data_ptr(), idx.data_ptr(), table.size, 1, 2, 0, 0, N, U.data_ptr(), o.data_ptr(), sb.data_ptr(), 0, ws, wsb, s)
host = (W.data_ptr(), idx.data_ptr(), table.size, 1, 2, 0, 0, N, U.data_ptr(), ho.data_ptr(), sb.data_ptr(), 0, ws, wsb, s)
clock("ctypes call, argument error (no launch)", lambda: L.dr_sample_dac(*bad))
clock("ctypes + cooperative launch", lambda: L.dr_sample_dac(*dev), 300)
clock("launch + sync, device out", lambda: (L.dr_sample_dac(*dev), L.dr_stream_synchronize(s)), 300)
clock("launch + sync, pinned out", lambda: (L.dr_sample_dac(*host), L.dr_stream_synchronize(s)), 300)
clock("launch + sync + memcpy d2h into pinned", lambda: (L.dr_sample_dac(*dev), ho.copy_(o, non_blocking=True),
                                                         L.dr_stream_synchronize(s)), 300)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for name, a in (("device out", dev), ("pinned out", host)):
    ts = []
    for _ in range(50):
        e0.record(); L.dr_sample_dac(*a); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1) * 1e3)
    print(f"{'kernel events, ' + name:48s} {np.median(ts):7.2f} us", flush=True)
clock("public dac_sampler host", lambda: drs.dac_sampler(table, N, drs.RngStream(5)), 300)
st = drs.RngStream(5)
clock("public dac_sampler host (one stream)", lambda: drs.dac_sampler(table, N, st), 300)

# fixed costs: a trivial torch kernel + stream sync, and a sync with nothing queued
x = torch.zeros(1, device="cuda")
clock("torch tiny kernel + synchronize", lambda: (x.add_(1), L.dr_stream_synchronize(s)), 1000)
clock("dr_stream_synchronize, idle stream", lambda: L.dr_stream_synchronize(s), 1000)
ev = torch.cuda.Event()
def ev_spin():
    L.dr_sample_dac(*dev)
    ev.record()
    while not ev.query():
        pass
clock("launch + event query spin, device out", ev_spin, 300)
