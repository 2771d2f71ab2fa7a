import sys, time
sys.path.insert(0, __import__("os").environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import numpy as np, torch
import paper_2604_01356_b200 as drs
from paper_2604_01356_b200 import _lib, samplers
from paper_2604_01356_b200._tensors import host_result_i64, finish_host
import bench
c = bench.CONFIGS["c3"]
table = drs.build_weight_table(bench.make_weights("c3"))
N = c["N"]; st = drs.RngStream(5)
L = _lib.lib()
def clock(name, fn, k=2000):
    for _ in range(20): fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(k): fn()
    dt = (time.perf_counter() - t0) / k * 1e6
    torch.cuda.synchronize()
    print(f"{name:40s} {dt:7.2f} us")
clock("stream_handle", _lib.stream_handle)
clock("lib()", _lib.lib)
clock("host_result_i64", lambda: host_result_i64(N))
s = _lib.stream_handle()
clock("_scratch_uniforms", lambda: samplers._scratch_uniforms(N, s))
clock("_status_buf", lambda: samplers._status_buf(s))
clock("workspace_bytes+workspace", lambda: _lib.workspace(_lib.workspace_bytes(_lib.OP_SORTED, N), s))
clock("_stream_args", lambda: samplers._stream_args(st, N + 1))
W = table.device_cum; U = samplers._scratch_uniforms(N, s); o = torch.empty(N, dtype=torch.int64, device="cuda"); sb = samplers._status_buf(s)
ws, wsb = _lib.workspace(_lib.workspace_bytes(_lib.OP_SORTED, N), s)
idx = table.device_index
args = (W.data_ptr(), idx.data_ptr(), table.size, 1, 2, 0, 0, N, U.data_ptr(), o.data_ptr(), sb.data_ptr(), 0, ws, wsb, s)
clock("data_ptr x5", lambda: (W.data_ptr(), idx.data_ptr(), U.data_ptr(), o.data_ptr(), sb.data_ptr()))
clock("dr_sample_dac ctypes (launch only)", lambda: L.dr_sample_dac(*args), 500)
clock("dr_stream_synchronize after launch", lambda: (L.dr_sample_dac(*args), L.dr_stream_synchronize(s)), 500)
clock("public dac_sampler device", lambda: drs.dac_sampler(table, N, st, device=True, out=o, uniforms_out=U), 500)
clock("public dac_sampler host", lambda: drs.dac_sampler(table, N, st), 500)
clock("public dac_sampler host, uniforms_out", lambda: drs.dac_sampler(table, N, st, uniforms_out=U), 500)
clock("torch.cuda.current_device", torch.cuda.current_device)
clock("_check_out(U)", lambda: samplers._check_out(U, N, torch.float64, "uniforms_out"))
pin = host_result_i64(N)
clock("launch + sync into one pinned buffer", lambda: (L.dr_sample_dac(W.data_ptr(), idx.data_ptr(), table.size, 1, 2, 0, 0, N, U.data_ptr(), pin.data_ptr(), sb.data_ptr(), 0, ws, wsb, s), L.dr_stream_synchronize(s)), 500)
ob = torch.empty(N, dtype=torch.int64, device="cuda")
clock("dr_sample_binary_dev ctypes (regular launch only)", lambda: L.dr_sample_binary_dev(W.data_ptr(), idx.data_ptr(), table.size, 1, 2, 0, 0, N, ob.data_ptr(), s), 500)
clock("dr_match_binary ctypes (pdl launch only)", lambda: L.dr_match_binary(W.data_ptr(), idx.data_ptr(), table.size, U.data_ptr(), N, ob.data_ptr(), s), 500)
clock("dr_version ctypes (no launch)", lambda: L.dr_version(), 2000)
