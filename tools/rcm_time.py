"""Time of the device RCM kernel sequence alone (config-2 pattern) versus the
host C++ RCM: python tools/rcm_time.py [k]"""
import ctypes
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1812_06160_b200 import _lib, device as dv, workloads as W
from paper_1812_06160_b200.csr import symmetrize_pattern

k = int(sys.argv[1]) if len(sys.argv) > 1 else 128
a = W.laplace7(k)
sym = symmetrize_pattern(a.pattern)
rs = np.ascontiguousarray(sym.row_start, dtype=np.int32)
col = np.ascontiguousarray(sym.col, dtype=np.int32)
n = a.n
d = dv.DevCsr.from_host(n, rs, col)
perm_d = dv.empty_i32(n)
nc = ctypes.c_int32(0)
lib = _lib.load()
for rep in range(2):
    torch.cuda.synchronize()
    t = time.perf_counter()
    rc = lib.jv_rcm_device(n, dv.ptr(d.row_start), dv.ptr(d.col), dv.ptr(perm_d), 64,
                           ctypes.byref(nc), dv.stream())
    torch.cuda.synchronize()
    td = time.perf_counter() - t
perm = np.empty(n, np.int32)
t = time.perf_counter()
lib.jv_rcm_host(n, rs.ctypes.data_as(ctypes.c_void_p), col.ctypes.data_as(ctypes.c_void_p),
                perm.ctypes.data_as(ctypes.c_void_p))
th = time.perf_counter() - t
print({"n": n, "device_s": round(td, 4), "host_s": round(th, 4), "rc": rc,
       "equal": bool(np.array_equal(dv.host_i64(perm_d, n), perm))})
