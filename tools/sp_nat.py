import sys, json, numpy as np, torch
sys.path.insert(0, '/root/repo')
from paper_1812_06160_b200 import workloads as W, device as dv
for name, a in [("c4_natural", W.stencil27(100)), ("c2_natural", W.laplace7(128))]:
    A = dv.DevCsr.from_host(a.n, a.row_start, a.col, a.val); A.tile_rows()
    x = dv.f64(np.random.default_rng(0).uniform(-1,1,a.n)); y = dv.empty_f64(a.n)
    for _ in range(3): dv.spmv_dev(A, x, y)
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(50): dv.spmv_dev(A, x, y)
    e1.record(); torch.cuda.synchronize()
    us = e0.elapsed_time(e1)/50*1e3
    b = 12*a.nnz + 20*a.n + 4
    print(json.dumps({"m": name, "us": us, "GBps": b/us/1e3}))
