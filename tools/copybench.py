"""Host<->device copy paths for the drop-in API (117 MB = config-2 values)."""
import time

import numpy as np
import torch

n = 14581760
a = np.random.default_rng(0).standard_normal(n)
d = torch.empty(n, dtype=torch.float64, device="cuda")
pin = torch.empty(n, dtype=torch.float64, pin_memory=True)
torch.cuda.synchronize()


def t(f, reps=5):
    f()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        f()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return min(ts) * 1e3


print("torch threads", torch.get_num_threads())
print("pageable H2D (from_numpy.to)      %.2f ms" % t(lambda: d.copy_(torch.from_numpy(a))))
print("host copy numpy->pinned (torch)   %.2f ms" % t(lambda: pin.copy_(torch.from_numpy(a))))
print("pinned H2D                         %.2f ms" % t(lambda: d.copy_(pin, non_blocking=True)))
print("pinned D2H                         %.2f ms" % t(lambda: pin.copy_(d, non_blocking=True)))
b = np.empty_like(a)
print("host copy pinned->numpy (np.copyto) %.2f ms" % t(lambda: np.copyto(b, pin.numpy())))
print("host copy pinned->numpy (torch)   %.2f ms" % t(lambda: torch.from_numpy(b).copy_(pin)))
print("pageable D2H (torch)              %.2f ms" % t(lambda: torch.from_numpy(b).copy_(d)))
cr = torch.cuda.cudart()


def reg():
    ptr = a.ctypes.data
    cr.cudaHostRegister(ptr, a.nbytes, 0)
    d.copy_(torch.from_numpy(a), non_blocking=True)
    torch.cuda.synchronize()
    cr.cudaHostUnregister(ptr)


print("hostRegister+H2D+unregister        %.2f ms" % t(reg))
