"""Host side of the CTA-resident region kernels (csrc/region.cu).

Thin wrappers over libjv's host C++ setup (csrc/regions_host.cpp): the
acyclic region partition of a factor pattern's lower DAG and the per-sweep
wave streams.  Pure host code (no device needed), so the plans are tested
on the CPU by replaying them (tests/test_region_plan.py).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib

KINDS = {"factor": 0, "fwd": 1, "bwd": 2}


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def partition(row_start, col, diag, nreg_max, max_rows=1 << 15, dims=0):
    """(nreg, region_of) of the lower DAG, or None when it does not fit.
    dims: topological orders refining the partition (3 boxes, 2 pencils;
    0 = up to 3)."""
    rs, cl, dg = _i32(row_start), _i32(col), _i32(diag)
    n = dg.size
    if n == 0:
        return None
    region_of = np.empty(n, np.int32)
    nreg = _lib.load().jv_region_partition_host(n, _p(rs), _p(cl), _p(dg), int(nreg_max),
                                                int(max_rows), int(dims), _p(region_of))
    return (int(nreg), region_of) if nreg > 0 else None


@dataclass
class WaveStream:
    kind: int
    nreg: int
    words: np.ndarray      # int32, 16-byte aligned wave blocks
    table: np.ndarray      # int32 [waves, 8] {block (16 B units), bytes, ring off, dyn off,
                           #  packed values (16 B units), bytes, packed vector (16 B units), bytes}
    sidx: np.ndarray       # int32 packed value -> position in val (-1: padding)
    vidx: np.ndarray       # int32 packed per-call vector -> row (-1: padding)
    reg_wave: np.ndarray   # int32 [nreg + 1]
    slot_ring: int         # in-region values ring (power of 2)
    max_waves: int
    S: int
    D: int
    CS: int
    CD: int
    remote_deps: int
    max_rows: int = 0        # most rows in one wave

    @property
    def waves(self):
        return self.table.shape[0]

    def smem_bytes(self):
        return int(_lib.load().jv_region_smem_fixed(self.slot_ring, self.max_waves)) + \
            self.CS + self.CD


def build_stream(sweep, row_start, col, diag, region_of, nreg, smem_budget, tau=0.0,
                 threads=None):
    """WaveStream of one sweep ("factor", "fwd", "bwd"), or None when a row
    does not qualify (factor: not stencil-class; solves: > 32 dependencies)
    or the plan does not fit in `smem_budget` bytes of shared memory.
    Without `threads`, waves of up to 512 rows are tried first and smaller
    ones when the rings would only allow a prefetch distance below 3."""
    if threads is None:
        # wider waves mean fewer barrier steps on the critical path: take the
        # widest that still prefetches >= 3 waves ahead
        best = None
        for t in (512, 256, 128):
            ws = _build(sweep, row_start, col, diag, region_of, nreg, smem_budget, tau, t)
            if ws is not None and (best is None or ws.D > best.D):
                best = ws
            if best is not None and best.D >= 3:
                break
        return best
    return _build(sweep, row_start, col, diag, region_of, nreg, smem_budget, tau, threads)


def _build(sweep, row_start, col, diag, region_of, nreg, smem_budget, tau, threads):
    lib = _lib.load()
    kind = KINDS[sweep]
    rs, cl, dg, ro = _i32(row_start), _i32(col), _i32(diag), _i32(region_of)
    threads = min(int(threads), lib.jv_region_threads())
    sizes = np.zeros(13, np.int64)
    h = lib.jv_rstream_build(kind, dg.size, _p(rs), _p(cl), _p(dg), _p(ro), int(nreg), threads,
                             int(smem_budget), int(tau > 0), _p(sizes))
    if h <= 0:
        return None
    words = np.empty(int(sizes[0]) // 4, np.int32)
    table = np.empty((int(sizes[1]), 8), np.int32)
    reg_wave = np.empty(int(nreg) + 1, np.int32)
    sidx = np.empty(max(int(sizes[10]), 1), np.int32)
    vidx = np.empty(max(int(sizes[11]), 1), np.int32)
    _lib.call("jv_rstream_export", ctypes.c_int64(h), _p(words), _p(table), _p(reg_wave), _p(sidx),
              _p(vidx))
    return WaveStream(kind, int(nreg), words, table, sidx[:int(sizes[10])], vidx[:int(sizes[11])],
                      reg_wave, int(sizes[3]),
                      int(sizes[4]), int(sizes[5]), int(sizes[6]), int(sizes[7]), int(sizes[8]), int(sizes[9]),
                      int(sizes[12]))


def records(ws: WaveStream, w):
    """(slot0, [record dicts]) of wave w (host decoding, for tests/tools)."""
    base = int(ws.table[w, 0]) * 4
    blk = ws.words[base:base + int(ws.table[w, 1]) // 4]
    cnt, slot0, K, NP = (int(x) for x in blk[:4])
    row, p0, meta = blk[4:4 + cnt], blk[4 + cnt:4 + 2 * cnt], blk[4 + 2 * cnt:4 + 3 * cnt]
    ref = blk[4 + 3 * cnt:4 + (3 + K) * cnt].reshape(K, cnt)
    off = 4 + (3 + K) * cnt
    pslot = blk[off:off + NP]
    out = []
    for i in range(cnt):
        nd = int(meta[i]) & 63
        refs = ref[:nd, i]
        out.append(dict(r=int(row[i]), p0=int(p0[i]), nd=nd, pub=(int(meta[i]) >> 6) & 1,
                        umask=(int(meta[i]) >> 7) & 15, refs=refs,
                        rsl=np.array([pslot[-1 - int(x)] for x in refs if x < 0], np.int64),
                        K=K, cnt=cnt, NP=NP))
    return slot0, out
