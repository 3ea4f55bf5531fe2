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


ONE_OFF = 144   # shared-memory offset of the constant 1.0 (region.cu)


def records(ws: WaveStream, w):
    """(slot0, [record dicts]) of wave w (host decoding, for tests/tools).
    refs are translated back from shared-memory byte offsets: >= 0 a slot of
    the region's value ring, < 0: -(1 + j), the wave's j-th remote
    dependency (mailbox slot pslot[j])."""
    base = int(ws.table[w, 0]) * 4
    blk = ws.words[base:base + int(ws.table[w, 1]) // 4]
    cnt, slot0, K, NP = (int(x) for x in blk[:4])
    rec = blk[4:4 + 8 * cnt].reshape(cnt, 8)
    kx = max(K - 4, 0)
    xref = blk[4 + 8 * cnt:4 + (8 + kx) * cnt].reshape(kx, cnt)
    off = 4 + (8 + kx) * cnt
    pslot = blk[off:off + NP]
    slot_base = 256 + 16 * ws.max_waves
    rem_base = slot_base + 8 * ws.slot_ring + ws.CS + int(ws.table[w, 3]) + int(ws.table[w, 5]) + \
        (int(ws.table[w, 7]) & 0xFFFF)

    def back(off):
        off = int(off)
        if slot_base <= off < slot_base + 8 * ws.slot_ring:
            assert (off - slot_base) % 8 == 0
            return (off - slot_base) // 8
        j = (off - rem_base) // 8
        assert (off - rem_base) % 8 == 0 and 0 <= j < NP, (off, rem_base, NP)
        return -1 - j

    out = []
    for i in range(cnt):
        meta = int(rec[i, 6])
        nd = meta & 63
        raw = [rec[i, k] if k < 4 else xref[k - 4, i] for k in range(nd)]
        assert all(int(rec[i, k]) == ONE_OFF for k in range(nd, 4))
        assert int(rec[i, 7]) == slot_base + 8 * ((slot0 + i) % ws.slot_ring)
        refs = np.array([back(x) for x in raw], np.int64)
        out.append(dict(r=int(rec[i, 5]), p0=int(rec[i, 4]), nd=nd, pub=(meta >> 6) & 1,
                        umask=(meta >> 7) & 15, refs=refs,
                        rsl=np.array([pslot[-1 - int(x)] for x in refs if x < 0], np.int64),
                        K=K, cnt=cnt, NP=NP))
    return slot0, out
