"""Where the streamed factor_serial's time goes (c2): host link alone in
each direction, both directions at once, the ticket factor per chunk, the
whole pipeline."""
import os, sys, time, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
from paper_1812_06160_b200 import device as dv, _lib

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
a, plan, s, blocks = bench.build_config(cfg)
ilu = plan.ilu
nnz = ilu.nnz
host = dv.host_f64(plan.assembled, nnz).copy()
assert dv.pinned_host(host)
out = np.empty_like(host)
assert dv.pinned_host(out)
dev = dv.empty_f64(nnz)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def t(fn, reps=5):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return sorted(ts)[len(ts) // 2] * 1e3


h2d = lambda st: _lib.call("jv_memcpy_async", dv.ptr(dev), ctypes.c_void_p(host.ctypes.data), 8 * nnz, 0, ctypes.c_void_p(st.cuda_stream))
d2h = lambda st: _lib.call("jv_memcpy_async", ctypes.c_void_p(out.ctypes.data), dv.ptr(dev), 8 * nnz, 1, ctypes.c_void_p(st.cuda_stream))
print("h2d_ms", t(lambda: h2d(s1)), "GB/s", 8 * nnz / t(lambda: h2d(s1)) / 1e6)
print("d2h_ms", t(lambda: d2h(s1)), "GB/s", 8 * nnz / t(lambda: d2h(s1)) / 1e6)
print("both_ms", t(lambda: (h2d(s1), d2h(s2))))
for k, ends in ((8, 0), (16, 0), (8, 2), (16, 2), (16, 3), (24, 3), (32, 4)):
    ilu.STREAM_CHUNKS = k
    ilu.STREAM_ENDS = ends
    ilu._chunk_cache = None
    f = lambda: (host.__setitem__(slice(None), dv.host_f64(plan.assembled, nnz)) if False else None, ilu.factor_streamed(host))
    # warm
    np.copyto(host, dv.host_f64(plan.assembled, nnz))
    ilu.factor_streamed(host)
    ts = []
    for _ in range(5):
        np.copyto(host, out if False else dv.host_f64(plan.assembled, nnz))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ilu.factor_streamed(host)
        ts.append(time.perf_counter() - t0)
    print("chunks", k, "ends", ends, "pipeline_ms", sorted(ts)[2] * 1e3)
# factor per chunk (device only)
ilu.STREAM_CHUNKS = 16
ilu.STREAM_ENDS = 0
ilu._chunk_cache = None
bounds, rs = ilu._chunks(16)
plan.reset_values()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(17)]
dv._lib.call("jv_reset_row", dv.ptr(ilu.err), dv.stream())
for c in range(16):
    ev[c].record()
    ilu._factor_tickets(int(bounds[c]), int(bounds[c + 1]), int(bounds[c]), False, reset=False)
ev[16].record()
torch.cuda.synchronize()
print("chunk factor us", [round(ev[c].elapsed_time(ev[c + 1]) * 1e3) for c in range(16)])
plan.reset_values()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record(); ilu._factor_tickets(0, ilu.n, 0, False); e1.record(); torch.cuda.synchronize()
print("full ticket factor us", e0.elapsed_time(e1) * 1e3)
