"""Host side of the hub-row gather plan (jv_hub_plan_host, csrc/host.cpp):
builds, for the largest heavy rows of a factor pattern, the target-parallel
schedule the factor kernel's gather path streams (setup; once per pattern).
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib


def plan_row(length, nL, piv_ptr, op_q, op_w, dslot):
    """Stream (int32 [m, 2]) and meta (int32) of one row; None if it does not fit."""
    nops = int(piv_ptr[nL] - piv_ptr[0])
    stream = np.empty(2 * (nops + nL) + 2, dtype=np.int32)
    meta = np.empty(1 + 33 * (nL + 2), dtype=np.int32)
    ns, nm = ctypes.c_int64(0), ctypes.c_int64(0)
    P = lambda a: a.ctypes.data_as(ctypes.c_void_p)
    piv_ptr = np.ascontiguousarray(piv_ptr, dtype=np.int64)
    op_q = np.ascontiguousarray(op_q, dtype=np.int32)
    op_w = np.ascontiguousarray(op_w, dtype=np.int32)
    dslot = np.ascontiguousarray(dslot, dtype=np.int32)
    rc = _lib.load().jv_hub_plan_host(int(length), int(nL), P(piv_ptr), P(op_q), P(op_w),
                                      P(dslot), P(stream), ctypes.byref(ns), P(meta),
                                      ctypes.byref(nm))
    if rc != 0:
        return None
    return stream[:2 * ns.value].reshape(-1, 2), meta[:nm.value]


def replay(stream, meta, av, nL, u_of, d_of):
    """Execute a plan exactly as the kernel's gather path does (lane by
    lane, step by step) on the row values `av` (modified in place):
    u_of(q) = value of U entry q of its pivot row, d_of(slot) = a pivot's
    diagonal.  Explicitly rounded: numpy float64 scalar ops."""
    nph = int(meta[0])
    base = 0
    for p in range(nph):
        qlen = meta[1 + 33 * p: 1 + 33 * p + 32]
        nfin = int(meta[1 + 33 * p + 32])
        cur = [-1] * 32
        acc = [0.0] * 32
        for t in range(int(qlen[0])):
            act = int(np.sum(qlen > t))
            for lane in range(act):
                x, y = int(stream[base + lane, 0]), int(stream[base + lane, 1])
                q, j, w = x & 0x7FFFFFFF, y & 0xFFFF, (y >> 16) & 0xFFFF
                if cur[lane] != w:
                    if cur[lane] >= 0:
                        av[cur[lane]] = acc[lane]
                    cur[lane] = w
                    acc[lane] = av[w]
                acc[lane] = np.float64(acc[lane]) - np.float64(av[j]) * np.float64(u_of(q))
            base += act
        for lane in range(32):
            if cur[lane] >= 0:
                av[cur[lane]] = acc[lane]
        for f in range(nfin):
            x, y = int(stream[base + f, 0]), int(stream[base + f, 1])
            w = (y >> 16) & 0xFFFF
            av[w] = np.float64(av[w]) / np.float64(d_of(x & 0x7FFFFFFF))
        base += nfin
    return av
