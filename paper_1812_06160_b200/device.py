"""Device-resident objects and the thin Python side of every libjv call.

PyTorch is used only for device memory, the current stream and small
index plumbing; all arithmetic of the hot path runs in libjv.so kernels.
Index arrays on the device are int32 (checked), values float64.
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field

import numpy as np

from . import _lib, regionplan
from ._lib import BackendUnavailable

_INT32_MAX = 2**31 - 1
_NO_ROW = _INT32_MAX

_torch = None


def torch():
    """Import torch lazily and require a CUDA device (no CPU fallback)."""
    global _torch
    if _torch is None:
        import torch as t

        _torch = t
    if not _torch.cuda.is_available():
        raise BackendUnavailable("no CUDA device: the ILU/stri/spmv path runs only on the GPU")
    _lib.load()
    return _torch


def _hp(a):
    """host numpy array -> ctypes pointer"""
    return a.ctypes.data_as(ctypes.c_void_p)


def stream():
    return ctypes.c_void_p(torch().cuda.current_stream().cuda_stream)


def ptr(t):
    return ctypes.c_void_p(0 if t is None else t.data_ptr())


def sync():
    torch().cuda.current_stream().synchronize()


def i32(a):
    """Host index array (any int dtype) -> device int32 tensor."""
    t = torch()
    a = np.asarray(a)
    if a.size and (a.max() > _INT32_MAX or a.min() < -_INT32_MAX):
        raise OverflowError("index values exceed int32; matrices need n, nnz < 2**31")
    return t.from_numpy(np.ascontiguousarray(a, dtype=np.int32)).to("cuda", non_blocking=False)


def f64(a):
    t = torch()
    return t.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to("cuda")


# ---- host <-> device transfers for the drop-in API ----------------------
# numpy arrays are pageable; a pinned staging buffer lets the DMA run at full
# link speed while torch's parallel host copy fills it chunk by chunk, so
# the host copy of chunk i+1 overlaps the DMA of chunk i.

_PIN = {}
_CHUNK = 1 << 21   # doubles per chunk (16 MB)


def _pinned(n):
    """The staging buffer, once its previous DMA has drained."""
    t = torch()
    ev = _PIN.get("busy")
    if ev is not None:
        ev.synchronize()
    buf = _PIN.get("f64")
    if buf is None or buf.numel() < n:
        buf = t.empty(max(n, 1), dtype=t.float64, pin_memory=True)
        _PIN["f64"] = buf
    return buf


def _mark_busy():
    ev = torch().cuda.Event()
    ev.record()
    _PIN["busy"] = ev


# Large numpy buffers handed to the API are page-locked in place once
# (cudaHostRegister) and then moved by DMA directly, without the staging
# copy; the registration is dropped when the array is garbage-collected.
_REG_MIN = 1 << 22     # bytes
_REGISTERED = {}       # data pointer -> nbytes


def _registered(a):
    """True when `a` (C-contiguous float64 numpy array) is page-locked."""
    if a.nbytes < _REG_MIN or not a.flags.c_contiguous or a.base is not None:
        return False
    p = a.ctypes.data
    if _REGISTERED.get(p) == a.nbytes:
        return True
    if p in _REGISTERED:
        return False
    if _lib.load().jv_host_register(ctypes.c_void_p(p), a.nbytes) != 0:
        _REGISTERED[p] = -1
        return False
    _REGISTERED[p] = a.nbytes
    import weakref

    def _release(p=p):
        _lib.load().jv_host_unregister(ctypes.c_void_p(p))
        _REGISTERED.pop(p, None)

    weakref.finalize(a, _release)
    return True


_REGION_D_CAP = int(os.environ.get("JV_REGION_D", "99"))   # diagnostics: shallower prefetch
STREAM_MIN_BYTES = 32 << 20    # streamed factor_serial above this many value bytes


def _is_registered(a):
    """True when `a` is already page-locked (never registers)."""
    return a.flags.c_contiguous and _REGISTERED.get(a.ctypes.data) == a.nbytes


def pinned_host(a):
    """Page-lock a float64 host array in place when possible (True if so)."""
    return isinstance(a, np.ndarray) and a.dtype == np.float64 and _registered(a)


VEC_CHUNK = 1 << 17   # doubles per staging chunk for vectors (1 MB)
_PIN_RESULT_MIN = 1 << 17   # doubles: results at least this long come back in pinned memory


def upload_f64(dst, src):
    """dst (device tensor) <- src (host float64 numpy array): whole value
    arrays (the residency tests and the bench count these calls)."""
    return _upload(dst, src, _CHUNK)


def _upload(dst, src, chunk, register=True):
    t = torch()
    if (isinstance(src, np.ndarray) and src.dtype == np.float64
            and (_registered(src) if register else _is_registered(src))):
        _lib.call("jv_memcpy_async", ptr(dst), ctypes.c_void_p(src.ctypes.data), src.nbytes, 0,
                  stream())
        sync()   # the caller may reuse its array as soon as we return
        return dst
    src = np.ascontiguousarray(src, dtype=np.float64)
    n = src.size
    if n == 0:
        return dst
    pin = _pinned(n)
    hsrc = t.from_numpy(src)
    for a in range(0, n, chunk):
        b = min(n, a + chunk)
        pin[a:b].copy_(hsrc[a:b])
        dst[a:b].copy_(pin[a:b], non_blocking=True)
    _mark_busy()
    return dst


def upload_vec(src, n):
    """New device vector <- host vector of length n (the per-call right-hand
    side of the drop-in solves): small staging chunks, so the host copy of
    one chunk runs beside the DMA of the previous one."""
    src = np.asarray(src, dtype=np.float64)
    if src.shape != (n,):
        raise ValueError(f"vector of shape {src.shape} for a system of {n} rows")
    x = empty_f64(n)
    # per-call vectors are usually fresh arrays: page-locking each one
    # (cudaHostRegister, ~ms) would cost more than the staging copy, so only
    # an array the caller already had registered takes the direct DMA
    _upload(x, src, VEC_CHUNK, register=False)
    return x


def download_vec(src, n):
    """Fresh host vector <- src[:n] (device).  Long results are written by
    one DMA straight into page-locked memory from torch's caching host
    allocator (the block goes back to the cache when the caller drops the
    array), so there is no staging copy and no first-touch page faulting."""
    t = torch()
    if n < _PIN_RESULT_MIN:
        return host_f64(src, n)
    out = t.empty(n, dtype=t.float64, pin_memory=True)
    out.copy_(src[:n], non_blocking=True)
    sync()
    return out.numpy()


def download_f64(dst, src, n=None):
    """dst (host float64 numpy array, written in place) <- src[:n] (device)."""
    t = torch()
    n = dst.size if n is None else n
    if n == 0:
        return dst
    if dst.dtype == np.float64 and _registered(dst):
        _lib.call("jv_memcpy_async", ctypes.c_void_p(dst.ctypes.data), ptr(src), 8 * n, 1,
                  stream())
        sync()
        return dst
    pin = _pinned(n)
    hdst = t.from_numpy(dst)
    events = []
    for a in range(0, n, _CHUNK):
        b = min(n, a + _CHUNK)
        pin[a:b].copy_(src[a:b], non_blocking=True)
        ev = t.cuda.Event()
        ev.record()
        events.append((a, b, ev))
    for a, b, ev in events:
        ev.synchronize()
        hdst[a:b].copy_(pin[a:b])
    return dst


def empty_i32(n):
    return torch().empty(max(int(n), 1), dtype=torch().int32, device="cuda")


def empty_f64(n):
    return torch().empty(max(int(n), 1), dtype=torch().float64, device="cuda")


def host_i64(t, n=None):
    a = t.cpu().numpy().astype(np.int64)
    return a if n is None else a[:n]


def host_f64(t, n=None):
    a = t.cpu().numpy().astype(np.float64)
    return a if n is None else a[:n]


class Mailbox:
    """Sync-free mailbox (16-byte packets or 8-byte words) plus its epoch.

    Epochs grow by one per kernel call, so stale packets from earlier calls
    never match; on 32-bit wrap the box is zeroed and the epoch restarts.
    """

    def __init__(self, slots, words_per_slot=2):
        self.words = words_per_slot
        self.slots = max(int(slots), 1)
        self.buf = torch().zeros(self.slots * words_per_slot, dtype=torch().int64, device="cuda")
        self.epoch = 0

    def next_epoch(self):
        self.epoch += 1
        if self.epoch >= 2**32 - 1:
            self.buf.zero_()
            self.epoch = 1
        return self.epoch

    def ensure(self, slots):
        if slots > self.slots:
            self.__init__(slots, self.words)
        return self


def reset_row_slot():
    slot = torch().empty(1, dtype=torch().int32, device="cuda")
    _lib.call("jv_reset_row", ptr(slot), stream())
    return slot


def read_row_slot(slot):
    """Host value of an error-row slot; -1 when no row was reported."""
    v = int(slot.item())
    return -1 if v == _NO_ROW else v


def check_hang():
    h = ctypes.c_int32(0)
    _lib.call("jv_status", ctypes.byref(h))
    if h.value:
        raise RuntimeError("a sync-free kernel wait timed out (schedule does not cover a dependency)")


# ------------------------------------------------------------- tail plan


# autotune candidate of the factorization: upper rows by the sync-free
# kernel, then the two-stage lower tail (csrc/tail.cu)
TWO_STAGE = {"two_stage": True, "nreg": 0}
# autotune candidate of every sweep of a small matrix: one CTA walks the
# levels with __syncthreads (csrc/cta.cu)
CTA = {"cta": True, "nreg": 0}
# autotune candidate of the solves of a small matrix: one thread block with
# the whole sweep in shared memory (jv_solve_small, csrc/solve.cu)
SMALL = {"small": True, "nreg": 0}
_CTA_MAX = []


def cta_max_rows():
    if not _CTA_MAX:
        _CTA_MAX.append(int(_lib.load().jv_cta_max_rows()))
    return _CTA_MAX[0]


class TailPlan:
    """Device plan of the lower tail (jv_tail_plan_build): update lists of
    stage 1 and the compact corner as its own DevIlu (structure only)."""

    def __init__(self, ilu, n_upper):
        import weakref
        lib = _lib.load()
        h = lib.jv_tail_plan_build(ilu.n, n_upper, ptr(ilu.row_start), ptr(ilu.col),
                                   ptr(ilu.diag_pos), int(ilu.milu), stream())
        if h <= 0:
            raise RuntimeError(f"jv_tail_plan_build failed ({h}): "
                               f"{lib.jv_last_error().decode(errors='replace')}")
        self.h = h
        self._fin = weakref.finalize(self, lib.jv_tail_plan_free, h)
        info = (ctypes.c_int64 * 6)()
        _lib.call("jv_tail_plan_info", h, info)
        self.nt, self.nl, self.nops, self.ngroups, self.nsegs, self.nc = (int(v) for v in info)
        self.n_upper = n_upper
        self.corner = None
        if self.nt:
            rs = empty_i32(self.nt + 1)
            col = empty_i32(self.nc)
            dg = empty_i32(self.nt)
            self.pos = empty_i32(self.nc)
            _lib.call("jv_tail_corner", h, ptr(rs), ptr(col), ptr(dg), ptr(self.pos), stream())
            self.crs = host_i64(rs, self.nt + 1)
            self.corner = DevIlu(self.nt, rs, col, dg)
            self.save = empty_f64(self.nc)


# ------------------------------------------------------------------ CSR


@dataclass
class DevCsr:
    """CSR resident in HBM: int32 structure, float64 values (or None)."""

    n: int
    nnz: int
    row_start: object
    col: object
    val: object = None
    _tile_rows: object = field(default=None, repr=False)

    @staticmethod
    def from_host(n, row_start, col, val=None):
        row_start = np.asarray(row_start)
        nnz = int(row_start[n]) if n else 0
        if nnz > _INT32_MAX:
            raise OverflowError("nnz exceeds int32")
        return DevCsr(
            int(n), nnz, i32(row_start), i32(col) if nnz else empty_i32(1),
            (f64(val) if nnz else empty_f64(1)) if val is not None else None,
        )

    def tile_rows(self):
        if self._tile_rows is None:
            tile = _lib.load().jv_spmv_tile()
            ntiles = max(1, -(-self.nnz // tile))
            self._tile_rows = empty_i32(2 * (ntiles + 1))
            _lib.call("jv_spmv_plan", self.n, self.nnz, ptr(self.row_start), ptr(self._tile_rows),
                      stream())
        return self._tile_rows

    def host_pattern(self):
        return host_i64(self.row_start, self.n + 1), host_i64(self.col, self.nnz)


def spmv_dev(a: DevCsr, x, y):
    """y = A x on the device (x, y float64 tensors of length n)."""
    _lib.call("jv_spmv", a.n, a.nnz, ptr(a.row_start), ptr(a.col), ptr(a.val), ptr(x), ptr(y),
              ptr(a.tile_rows()), stream())
    return y


# ----------------------------------------------------------- level sets


def levels_dev(a: DevCsr, backward: bool):
    """Longest-path levels (int32 tensor) and the level count."""
    level_of = empty_i32(a.n)
    box = Mailbox(a.n, 1)
    nlev = ctypes.c_int32(0)
    _lib.call("jv_levels", int(backward), a.n, ptr(a.row_start), ptr(a.col), ptr(level_of),
              ptr(box.buf), box.next_epoch(), ctypes.byref(nlev), stream())
    check_hang()
    return level_of, int(nlev.value)


def level_sort_dev(n, nlev, level_of):
    order = empty_i32(n)
    level_ptr = empty_i32(nlev + 1)
    _lib.call("jv_level_sort", n, nlev, ptr(level_of), ptr(order), ptr(level_ptr), stream())
    return order, level_ptr


def batches_dev(nlev, level_ptr, n):
    batch_ptr = empty_i32(n // 32 + nlev + 2)
    nb = ctypes.c_int32(0)
    _lib.call("jv_build_batches", nlev, ptr(level_ptr), ptr(batch_ptr), ctypes.byref(nb), stream())
    return batch_ptr, int(nb.value)


@dataclass
class Schedule:
    """Level-batched row order for a sync-free sweep (jv_build_schedule_n):
    keys = nclass*level + class; class c rows steps[c] per batch."""

    order: object
    batch_ptr: object
    nbatch: int
    nkeys: int
    keys: object = None      # per-row key (indexed by row id)
    steps: tuple = (32, 1)

    def restrict(self, lo, hi):
        """Rows with lo <= index < hi, keeping level order and classes."""
        t = torch()
        rows = t.arange(lo, hi, dtype=t.int32, device="cuda")
        keys = self.keys[lo:hi].contiguous()
        sub = build_schedule(rows, keys, self.nkeys, self.steps)
        sub.keys = self.keys
        return sub

    def batch_class(self):
        """int8 class of every batch (key % nclass of its first row)."""
        if getattr(self, "_bclass", None) is None:
            t = torch()
            first = self.order[self.batch_ptr[:self.nbatch].long()].long()
            self._bclass = (self.keys[first] % len(self.steps)).to(t.int8).contiguous()
        return self._bclass


def build_schedule(rows, keys, nkeys, steps=(32, 1)):
    m = int(keys.numel())
    order = empty_i32(m)
    batch_ptr = empty_i32(m + nkeys + 2)
    nb = ctypes.c_int32(0)
    st = (ctypes.c_int32 * len(steps))(*steps)
    _lib.call("jv_build_schedule_n", m, ptr(rows), ptr(keys), int(nkeys), len(steps), st,
              ptr(order), ptr(batch_ptr), ctypes.byref(nb), stream())
    return Schedule(order, batch_ptr, int(nb.value), nkeys, None, tuple(steps))


def schedule_dev(a: DevCsr, backward: bool, cls=None, steps=(32, 1), level_of=None):
    """Schedule of a sweep over pattern `a`: its levels (forward: columns <
    r, backward: columns > r) plus per-row classes (None = all class 0)."""
    t = torch()
    if level_of is None:
        level_of, nlev = levels_dev(a, backward)
    else:
        nlev = int(level_of.max().item()) + 1 if level_of.numel() else 0
    nclass = len(steps)
    keys = level_of.to(t.int32) * nclass
    if cls is not None:
        keys = keys + cls
    keys = keys.contiguous()
    sched = build_schedule(None, keys, nclass * max(nlev, 1), steps)
    sched.keys = keys
    return sched, level_of


# --------------------------------------------------------- ILU factors


class DevIlu:
    """Factor storage resident in HBM plus the schedules of its three sweeps.

    factor(): sync-free ILU(k, tau) in place on `val`;
    solve(which, b, out): forward (unit L) / backward (U) sweeps.
    """

    def __init__(self, n, row_start, col, diag_pos, val=None, tau=0.0, milu=False):
        self.n = int(n)
        self.row_start = row_start
        self.col = col
        self.diag_pos = diag_pos
        self.nnz = int(row_start[self.n].item()) if self.n else 0
        self.val = val if val is not None else empty_f64(self.nnz)
        self.tau = float(tau)
        self.milu = bool(milu)
        self.pattern = DevCsr(self.n, self.nnz, row_start, col)
        self._fwd = None
        self._bwd = None
        self._fsched = None
        self._fsched_milu = None
        self._regions = None
        self._rstreams = {}
        self._rchoice = {}
        self.autotune_ms = {}
        self._hpat = None
        self._vver = 0
        self._csrls = {}
        self._side = None
        self._sms = None
        self._elim = None
        self._fwd_levels = None
        self.holder = None      # whose values `val` holds (IluFactors / IluPreconditioner)
        self.n_upper = None     # first lower-tail row (set by the device plan)
        self.norms = empty_f64(self.n)
        self.fbox = Mailbox(self.nnz, 2)
        self.sbox = Mailbox(self.n, 2)
        self.err = reset_row_slot()
        # batch tickets of the factor and solve kernels (kernels leave them 0)
        self.ticket = torch().zeros(4, dtype=torch().int32, device="cuda")

    @staticmethod
    def from_host(n, row_start, col, diag_pos, val, tau=0.0, milu=False):
        return DevIlu(n, i32(row_start), i32(col) if len(col) else empty_i32(1),
                      i32(diag_pos) if n else empty_i32(1), f64(val) if len(val) else empty_f64(1),
                      tau, milu)

    # schedules --------------------------------------------------------
    def _factor_classes(self):
        key = bool(self.milu)
        if getattr(self, "_fcls", None) is None or self._fcls[0] != key:
            self._fcls = (key, self._classes("factor"))
        return self._fcls[1]

    def _classes(self, kind):
        cls = empty_i32(self.n)
        if kind == "factor":
            _lib.call("jv_classify_factor", self.n, ptr(self.row_start), ptr(self.col),
                      ptr(self.diag_pos), int(self.milu), ptr(cls), stream())
        else:
            _lib.call("jv_classify_solve", 0 if kind == "fwd" else 1, self.n,
                      ptr(self.row_start), ptr(self.diag_pos), ptr(cls), stream())
        return cls

    def factor_schedule(self):
        """Factor sweep schedule: thread-path rows 32 to a batch, pairable
        listed warp rows (jv_elim_lists flag 1) two to a batch, other warp
        rows one to a batch."""
        if self._fsched is None or self._fsched_milu != self.milu:
            t = torch()
            cls = self._factor_classes()
            el = self.elim_lists()
            cls3 = cls
            if el is not None:
                flags = el[0][:self.n].to(t.int32)
                cls3 = t.where(cls == 0, t.zeros_like(cls),
                               t.where(flags == 1, t.ones_like(cls), t.full_like(cls, 2)))
            else:
                cls3 = cls * 2
            self._fsched, self._fwd_levels = schedule_dev(self.pattern, False,
                                                          cls3.to(t.int32).contiguous(),
                                                          steps=(self.THREAD_BATCH, 2, 1),
                                                          level_of=self._fwd_levels)
            self._fsched_milu = self.milu
        return self._fsched

    # heavy rows: structural matches precomputed once per pattern (jv_elim_lists)
    ELIM_MIN_CAND = 256
    THREAD_BATCH = 32         # thread-path rows per factor batch (24/16/8 measured no better)
    ELIM_WARP_ROWS = True     # lists for every warp-path row, not only heavy ones

    def elim_lists(self):
        """(heavy, elim_ptr, elim) device buffers, or None if no row is heavy."""
        key = bool(self.milu)
        if self._elim is None or self._elim[0] != key:
            t = torch()
            heavy = t.empty(max(self.n, 1), dtype=t.int8, device="cuda")
            eptr = t.empty(self.nnz + 1, dtype=t.int64, device="cuda")
            nops = ctypes.c_int64(0)
            args = [self.n, ptr(self.row_start), ptr(self.col), ptr(self.diag_pos), int(self.milu),
                    self.ELIM_MIN_CAND, ptr(self._factor_classes()) if self.ELIM_WARP_ROWS else None,
                    ptr(heavy), ptr(eptr)]
            _lib.call("jv_elim_lists", *args, None, ctypes.byref(nops), stream())
            lists = None
            if nops.value > 0:
                elim = t.empty(2 * nops.value, dtype=t.int32, device="cuda")
                _lib.call("jv_elim_lists", *args, ptr(elim), ctypes.byref(nops), stream())
                lists = (heavy, eptr, elim, int(nops.value))
            self._elim = (key, lists)
        return self._elim[1]

    # hub rows: target-parallel gather plans (jv_hub_plan_host) for the
    # heavy rows with at least HUB_MIN_OPS updates
    HUB_MIN_OPS = 1024

    def hub_plans(self):
        """(stream, sptr, meta, mptr) device buffers or None; flags the
        planned rows 4 in the elimination-list flags."""
        el = self.elim_lists()
        if el is None or self.milu:      # MILU lists carry out-of-pattern targets
            return None
        if getattr(self, "_hub", None) is not None and self._hub[0] is el:
            return self._hub[1]
        from concurrent.futures import ThreadPoolExecutor
        from . import hubplan
        t = torch()
        n = self.n
        flags_d, eptr_d, elim_d = el[0], el[1], el[2]
        flags = flags_d[:n].cpu().numpy()
        rs = host_i64(self.row_start, n + 1)
        dg = host_i64(self.diag_pos, n)
        cand = np.flatnonzero(flags == 2)
        plans = None
        if cand.size:
            e_rs = eptr_d[t.from_numpy(rs[cand]).cuda()].cpu().numpy()
            e_dg = eptr_d[t.from_numpy(dg[cand]).cuda()].cpu().numpy()
            sel = cand[(e_dg - e_rs) >= self.HUB_MIN_OPS]
            if sel.size:
                def one(r):
                    L = int(dg[r] - rs[r])
                    piv = eptr_d[int(rs[r]):int(rs[r]) + L + 1].cpu().numpy()
                    ops = elim_d[2 * int(piv[0]):2 * int(piv[-1])].cpu().numpy().reshape(-1, 2)
                    cols = self.col[int(rs[r]):int(rs[r]) + L].long()
                    dslot = self.diag_pos[cols].cpu().numpy()
                    return hubplan.plan_row(int(rs[r + 1] - rs[r]), L, piv, ops[:, 0], ops[:, 1],
                                            dslot)
                with ThreadPoolExecutor(8) as ex:
                    out = list(ex.map(one, sel))
                keep = [(r, pl) for r, pl in zip(sel, out) if pl is not None]
                if keep:
                    sptr = np.full(n, -1, np.int64)
                    mptr = np.full(n, -1, np.int64)
                    so = mo = 0
                    for r, (st, me) in keep:
                        sptr[r], mptr[r] = so, mo
                        so += st.shape[0]
                        mo += me.size
                    stream = np.concatenate([st for _, (st, _) in keep]).astype(np.int32)
                    meta = np.concatenate([me for _, (_, me) in keep]).astype(np.int32)
                    rows = t.from_numpy(np.array([r for r, _ in keep], np.int64)).cuda()
                    flags_d[rows] = 4
                    plans = (t.from_numpy(stream.reshape(-1)).cuda(), t.from_numpy(sptr).cuda(),
                             t.from_numpy(meta).cuda(), t.from_numpy(mptr).cuda(), len(keep))
        self._hub = (el, plans)
        return plans

    def fwd_schedule(self):
        if self._fwd is None:
            self._fwd, _ = schedule_dev(self.pattern, False, self._classes("fwd"))
        return self._fwd

    def bwd_schedule(self):
        if self._bwd is None:
            self._bwd, _ = schedule_dev(self.pattern, True, self._classes("bwd"))
        return self._bwd

    # numerics ---------------------------------------------------------
    def compute_norms(self):
        _lib.call("jv_row_norms", self.n, ptr(self.row_start), ptr(self.val), self.tau,
                  ptr(self.norms), stream())

    # CTA-resident region kernels ------------------------------------------
    # One co-resident CTA per region of an acyclic box-like partition of the
    # lower DAG (jv_region_partition_host); per sweep a wave stream
    # (jv_rstream_build).  The factorization takes this path for
    # stencil-class matrices (<= 4 pivots, pivots' U rows meeting the row
    # only at its diagonal, no MILU), the solves for rows with <= 32
    # dependencies; everything else runs the ticket kernels.  Both paths give
    # the same bits.  JV_REGIONS=0 (or use_regions = False) turns it off.
    # "auto": each sweep takes the faster of the two paths, timed once on
    # first use (both give the same bits); "on" / "off" force it
    region_mode = {"0": "off", "1": "on"}.get(os.environ.get("JV_REGIONS", ""), "auto")

    @property
    def use_regions(self):
        return self.region_mode != "off"

    @use_regions.setter
    def use_regions(self, on):
        self.region_mode = "on" if on else "off"

    def _region_for(self, sweep):
        """The region stream when the region path runs this sweep, else None."""
        if not self.use_regions:
            return None
        if self.region_mode == "on":
            return self.region_stream(sweep)
        key = (sweep, sweep == "factor" and self.tau > 0)
        if key not in self._rchoice:
            self._rchoice[key] = self._autotune(sweep)
        return self._rchoice[key]

    def _autotune(self, sweep):
        """Time the ticket kernel and every region-plan candidate of one sweep
        once each (after a warm-up launch); keep the fastest (all give the
        same bits) and free the other plans."""
        t = torch()
        cands = [None]
        for c in self.region_candidates.get(sweep, [(0, 0)]):
            rp = self._stream_for(sweep, c)
            if rp is not None and all(rp is not x for x in cands):
                cands.append(rp)
        if sweep == "factor" and self.n_upper is not None and 0 < self.n_upper < self.n:
            cands.append(TWO_STAGE)
        if 0 < self.n <= cta_max_rows() and self.cta_ok(sweep):
            cands.append(CTA)
        if sweep != "factor" and self._small_plan(0 if sweep == "fwd" else 1) is not None:
            cands.append(SMALL)
        if len(cands) == 1:
            self.autotune_ms[sweep] = ()
            return None
        ev = [t.cuda.Event(enable_timing=True) for _ in range(4)]
        if sweep == "factor":
            save = self.val.clone()
        else:
            which = 0 if sweep == "fwd" else 1
            vin = t.ones(self.n, dtype=t.float64, device="cuda")
            vout = t.empty_like(vin)

        def run(rp):
            if sweep == "factor":
                if rp is None:
                    self._factor_tickets(0, self.n, 0, True)
                elif rp is TWO_STAGE:
                    self.factor_two_stage_async(self.n_upper)
                elif rp is CTA:
                    self._factor_cta(True)
                else:
                    self._factor_region(rp, True)
            elif rp is None:
                self._solve_tickets(which, vin, vout)
            elif rp is CTA:
                self._solve_cta(which, vin, vout)
            elif rp is SMALL:
                self._solve_small(which, vin, vout)
            else:
                self._region_run(rp, 1 + which, vin, vout, self.sbox)

        times = []
        for rp in cands:          # one warm-up launch, then the best of three
            best = float("inf")
            for rep in range(4):
                if sweep == "factor":
                    self.val.copy_(save)
                    self.values_changed()
                ev[0].record()
                run(rp)
                ev[1].record()
                t.cuda.synchronize()
                if rep:
                    best = min(best, ev[0].elapsed_time(ev[1]))
            times.append(best)
        if sweep == "factor":
            self.val.copy_(save)
            self.values_changed()
            _lib.call("jv_reset_row", ptr(self.err), stream())
        check_hang()
        # a region plan also costs its per-factorization value pack, not in
        # these timings: it has to win by a margin
        k = int(np.argmin(times))
        best = cands[k] if times[k] < 0.97 * times[0] else None
        self.autotune_ms[sweep] = tuple(times)
        for k in [k for k, v in self._rstreams.items() if k[0] == sweep and v is not best
                  and v is not TWO_STAGE and v is not CTA and v is not SMALL]:
            del self._rstreams[k]   # free the losing plans
        return best

    region_min_rows = 64
    region_max_rows = 1 << 22   # larger matrices (config 5's 16.7 M-row batch) keep the tickets
    region_single_max = 32768   # rows: up to here one region (one CTA) holds the matrix
    region_hint = None
    KIND = {"factor": 0, "fwd": 1, "bwd": 2}

    def set_regions(self, region_of):
        """Caller-supplied partition: region id per row (factor numbering),
        ids 0..R-1 with R <= #SMs (e.g. an application's domain decomposition)."""
        self.region_hint = np.ascontiguousarray(region_of, dtype=np.int32)
        self._regions = None
        self._rstreams = {}
        self._rchoice = {}

    def _host_pattern(self):
        if self._hpat is None:
            n = self.n
            host = lambda x, m: np.ascontiguousarray(x[:m].cpu().numpy(), dtype=np.int32)
            self._hpat = (host(self.row_start, n + 1), host(self.col, self.nnz),
                          host(self.diag_pos, n))
        return self._hpat

    # topological orders refining each sweep's partition (3: boxes, 2:
    # pencils); measured on config 2 the factorization prefers pencils
    # region-plan candidates per sweep: (partition orders: 3 boxes, 2
    # pencils; region cap, 0 = one per SM).  "on" uses the first; "auto"
    # times all of them against the ticket kernel (measured: config 2's
    # factor prefers 144 pencils, its solves 64 pencils; config 3 100 boxes,
    # config 4 144 boxes)
    region_candidates = {"factor": [(2, 0), (3, 0), (2, 64)],
                         "fwd": [(3, 0), (2, 64), (3, 100), (2, 0)],
                         "bwd": [(3, 0), (2, 64), (3, 100), (2, 0)]}

    def regions(self, dims=0, rmax=0):
        """(nreg, region_of) or None."""
        if self._regions is None:
            self._regions = {}
        if (dims, rmax) not in self._regions:
            self._regions[(dims, rmax)] = self._partition(dims, rmax) or False
        return self._regions[(dims, rmax)] or None

    def _partition(self, dims=0, rmax=0):
        if self.region_hint is not None:
            return int(self.region_hint.max()) + 1, self.region_hint
        rs, col, diag = self._host_pattern()
        t = torch()
        sms = t.cuda.get_device_properties(t.cuda.current_device()).multi_processor_count
        # a small matrix fits one CTA: no cross-region hops at all
        nreg = 1 if self.n <= self.region_single_max else min(sms, rmax or sms)
        return regionplan.partition(rs, col, diag, nreg, max_rows=1 << 20, dims=dims)

    def region_stream(self, sweep):
        """Device wave stream of one sweep ("factor", "fwd", "bwd") or None
        when the region path does not apply: the autotuned plan if the
        sweep was tuned, else the first candidate."""
        if not self.use_regions:
            return None
        key = (sweep, sweep == "factor" and self.tau > 0)
        if key in self._rchoice:
            return self._rchoice[key]
        return self._stream_for(sweep, self.region_candidates.get(sweep, [(0, 0)])[0])

    def _stream_for(self, sweep, cand):
        key = (sweep, cand, sweep == "factor" and self.tau > 0)
        if key not in self._rstreams:
            self._rstreams[key] = self._build_rstream(sweep, cand) or False
        return self._rstreams[key] or None

    def _build_rstream(self, sweep, cand=(0, 0)):
        if self.n < self.region_min_rows or self.n > self.region_max_rows:
            return None
        if sweep == "factor" and self.milu:
            return None
        reg = self.regions(*cand)
        if reg is None:
            return None
        nreg, region_of = reg
        rs, col, diag = self._host_pattern()
        t = torch()
        props = t.cuda.get_device_properties(t.cuda.current_device())
        budget = props.shared_memory_per_block_optin - 2048   # static shared memory headroom
        ws = regionplan.build_stream(sweep, rs, col, diag, region_of, nreg, budget, self.tau)
        if ws is None:
            return None
        up = lambda a: t.from_numpy(np.ascontiguousarray(a)).to("cuda")
        m, mv = int(ws.sidx.size), int(ws.vidx.size)
        return dict(nreg=nreg, words=up(ws.words), table=up(ws.table), reg_wave=up(ws.reg_wave),
                    sidx=up(ws.sidx) if m else None, m=m,
                    pack=t.empty(max(m, 2), dtype=t.float64, device="cuda"), pver=-1,
                    vidx=up(ws.vidx) if mv else None, mv=mv,
                    vpack=t.empty(max(mv, 2), dtype=t.float64, device="cuda"),
                    slot_ring=ws.slot_ring, max_waves=ws.max_waves, S=ws.S, D=ws.D, CS=ws.CS,
                    CD=ws.CD, waves=ws.waves, remote_deps=ws.remote_deps, max_rows=ws.max_rows,
                    kmax=int(ws.words[ws.table[:, 0].astype(np.int64) * 4 + 2].max()))

    def values_changed(self):
        """Invalidate the wave-ordered value copies (call after writing val)."""
        self._vver += 1

    def _pack(self, rp):
        """Refresh the sweep's wave-ordered copy of the matrix values."""
        if rp["pver"] != self._vver:
            _lib.call("jv_pack_values", rp["m"], ptr(rp["sidx"]), ptr(self.val), ptr(rp["pack"]),
                      stream())
            rp["pver"] = self._vver

    def _side_pack(self, rp, src=None):
        """Refresh `rp`'s value pack (from `src`, default the values) on a
        side stream that starts where the current stream is now; returns the
        event the current stream must wait on before anything that reads the
        pack or writes the source."""
        t = torch()
        if self._side is None:
            self._side = t.cuda.Stream()
        self._side.wait_stream(t.cuda.current_stream())
        src = self.val if src is None else src
        _lib.call("jv_pack_values", rp["m"], ptr(rp["sidx"]), ptr(src), ptr(rp["pack"]),
                  self._side.cuda_stream)
        rp["pver"] = self._vver
        ev = t.cuda.Event()
        ev.record(self._side)
        return ev

    def load_values(self, src):
        """values <- `src` (a device copy of the same pattern's values, e.g.
        the assembled matrix for a refactorization).  (Gathering the
        factorization's value pack from `src` on a side stream during the
        copy was measured: no gain, both are bandwidth-bound.)"""
        self.val.copy_(src)
        self.values_changed()

    def _region_run(self, rp, kind, inp, out, box, before_kernel=None, reset=None):
        # one launch in front of the sweep: its value pack when stale, the
        # per-call vector pack, the error-row reset
        m1 = 0
        if rp["pver"] != self._vver:
            m1 = rp["m"]
            rp["pver"] = self._vver
        m2 = rp["mv"]
        vsrc = (inp if kind != 0 else self.norms) if m2 else None
        if m1 or m2 or reset is not None:
            _lib.call("jv_pack_values2", m1, ptr(rp["sidx"]), ptr(self.val), ptr(rp["pack"]),
                      m2, ptr(rp["vidx"]) if m2 else None, ptr(vsrc), ptr(rp["vpack"]) if m2 else None,
                      ptr(reset), stream())
        if before_kernel is not None:
            before_kernel()
        _lib.call("jv_region_run", kind, rp["nreg"], rp["max_rows"] | (rp["kmax"] << 16), ptr(rp["words"]),
                  ptr(rp["table"]),
                  ptr(rp["reg_wave"]), rp["slot_ring"], rp["max_waves"], rp["S"],
                  min(rp["D"], _REGION_D_CAP),
                  rp["CS"], rp["CD"], ptr(self.val), ptr(rp["pack"]), ptr(rp["vpack"]),
                  ptr(out), ptr(self.norms),
                  self.tau, ptr(box.buf), box.next_epoch(), ptr(self.err), stream())

    def factor_async(self, lo=0, hi=None, ready_below=0, norms=True):
        """Launch the factorization of rows [lo, hi) (all by default)."""
        hi = self.n if hi is None else hi
        if lo == 0 and hi == self.n and ready_below == 0:
            rp = self._region_for("factor")
            if rp is TWO_STAGE:
                self.factor_two_stage_async(self.n_upper)
                return
            if rp is CTA:
                self._factor_cta(norms)
                self.values_changed()
                return
            if rp is not None:
                self._factor_region(rp, norms)
                self.values_changed()
                return
        self._factor_tickets(lo, hi, ready_below, norms)
        self.values_changed()

    def _factor_region(self, rp, norms):
        if norms and self.tau > 0:
            self.compute_norms()
        self._region_run(rp, 0, None, None, self.fbox, reset=self.err)

    def _factor_tickets(self, lo, hi, ready_below, norms, reset=True):
        sched = self.factor_schedule()
        el = self.elim_lists()
        hub = self.hub_plans()
        if lo > 0 or hi < self.n:
            if getattr(self, "_sub", None) is None or self._sub[0] is not sched:
                self._sub = (sched, {})
            key = (lo, hi)
            if key not in self._sub[1]:
                self._sub[1][key] = sched.restrict(lo, hi)
            sched = self._sub[1][key]
        if norms:
            self.compute_norms()
        if reset:
            _lib.call("jv_reset_row", ptr(self.err), stream())
        _lib.call("jv_factor", self.n, ptr(self.row_start), ptr(self.col), ptr(self.val),
                  ptr(self.diag_pos), ptr(self.norms), self.tau, int(self.milu), ptr(sched.order),
                  ptr(sched.batch_ptr), sched.nbatch, int(ready_below), ptr(self.fbox.buf),
                  self.fbox.next_epoch(), ptr(self.err), ptr(self.ticket),
                  ptr(el[0]) if el else None, ptr(el[1]) if el else None,
                  ptr(el[2]) if el else None,
                  ptr(sched.batch_class()) if sched.nbatch else None,
                  *([ptr(x) for x in hub[:4]] if hub else [None] * 4), stream())

    # lower-tail two-stage factorization (csrc/tail.cu) ----------------
    def tail_plan(self, n_upper):
        """Plan of the lower tail rows [n_upper, n) (cached per n_upper and
        MILU flag): stage-1 update lists and the compact corner."""
        key = (int(n_upper), bool(self.milu))
        if getattr(self, "_tail", None) is None or self._tail[0] != key:
            self._tail = (key, TailPlan(self, int(n_upper)))
        return self._tail[1]

    def factor_tail_async(self, n_upper, norms=True, ev=None):
        """Two-stage lower tail (lower.py:273-318): stage 1 eliminates every
        tail row's upper-stage pivots (jv_tail_upper, segmented, one warp
        per row), stage 2 factors the corner with the sync-free kernel on
        its compact copy and scatters it back.  Rows < n_upper must be
        factored.  The corner's error slot holds the corner row (or none)."""
        tp = self.tail_plan(n_upper)
        if tp.nt == 0:
            return tp
        if norms and self.tau > 0:
            self.compute_norms()
        if ev is not None:
            ev[0].record()
        _lib.call("jv_tail_upper", tp.h, ptr(self.col), ptr(self.diag_pos), ptr(self.val),
                  ptr(self.norms), self.tau, stream())
        if ev is not None:
            ev[1].record()
        c = tp.corner
        c.tau, c.milu = self.tau, self.milu
        # the corner's path (sync-free tickets or one CTA walking its
        # levels) is timed once on its first use, before any value moves
        mode = c._region_for("factor") if c.region_mode == "auto" else None
        if tp.nc:
            _lib.call("jv_gather", tp.nc, ptr(tp.pos), ptr(self.val), ptr(c.val), stream())
            tp.save.copy_(c.val[:tp.nc])
        c.values_changed()
        if self.tau > 0:
            c.norms[:tp.nt].copy_(self.norms[n_upper:self.n])
        if mode is CTA:
            c._factor_cta(False)
        else:
            c._factor_tickets(0, tp.nt, 0, False)
        if tp.nc:
            _lib.call("jv_scatter", tp.nc, ptr(tp.pos), ptr(c.val), ptr(self.val), stream())
        if ev is not None:
            ev[2].record()
        self.values_changed()
        return tp

    def factor_tail(self, n_upper):
        """factor_tail_async + the reference's error semantics: the smallest
        zero-pivot row (or -1); rows after it keep their stage-1 values, as
        the serial corner kernel stops there (_kernels.py:231-240)."""
        tp = self.factor_tail_async(n_upper)
        if tp.nt == 0:
            return -1
        bad = read_row_slot(tp.corner.err)
        check_hang()
        if bad < 0:
            return -1
        k = int(tp.crs[bad + 1])
        if k < tp.nc:
            _lib.call("jv_scatter", tp.nc - k, ctypes.c_void_p(tp.pos.data_ptr() + 4 * k),
                      ctypes.c_void_p(tp.save.data_ptr() + 8 * k), ptr(self.val), stream())
        self.values_changed()
        return n_upper + bad

    def factor_two_stage_async(self, n_upper, ev=None):
        """Upper rows with the sync-free kernel, then the lower tail
        (ev: 3 events recorded before stage 1, after it, after the corner)."""
        if n_upper > 0:
            self._factor_tickets(0, n_upper, 0, True)
        self.factor_tail_async(n_upper, norms=(n_upper == 0), ev=ev)
        self.values_changed()

    # single-CTA level-synchronous kernels (csrc/cta.cu) -----------------
    CTA_RINGS = (5, 4, 3, 2)    # row-data ring depths tried, deepest first
    CTA_MAX_PROGRAM = 1 << 26   # ints of level programs worth building

    def cta_programs(self):
        """Level programs of the single-CTA kernels per sweep ("factor",
        "fwd", "bwd") -> dict(prog, lbase, nlev, maxblk, maxstage, resident)
        or None when that sweep does not fit one CTA (cached per MILU)."""
        key = bool(self.milu)
        if getattr(self, "_cta", None) is not None and self._cta[0] == key:
            return self._cta[1]
        lib = _lib.load()
        t = torch()
        out = {"factor": None, "fwd": None, "bwd": None}
        if 0 < self.n <= cta_max_rows():
            h = lib.jv_cta_plan_build(self.n, ptr(self.row_start), ptr(self.col),
                                      ptr(self.diag_pos), int(self.milu), stream())
            if h <= 0:
                raise RuntimeError(f"jv_cta_plan_build failed ({h}): "
                                   f"{lib.jv_last_error().decode(errors='replace')}")
            try:
                out = self._cta_build(lib, h)
            finally:
                lib.jv_cta_plan_free(h)
        self._cta = (key, out)
        return out

    def _cta_build(self, lib, h):
        """Host-side program build from the device update lists (setup)."""
        t = torch()
        rs, col, dg = (np.ascontiguousarray(x) for x in self._host_pattern())
        n, nnz = self.n, self.nnz
        lens = rs[1:].astype(np.int64) - rs[:-1]
        nL = dg.astype(np.int64) - rs[:-1]
        # the device plan's lists, copied back once (small matrices only)
        if self._fwd_levels is None:
            self._fwd_levels, _ = levels_dev(self.pattern, False)
        out = {}
        bl, nb = levels_dev(self.pattern, True)
        self._cta_nofactor = False
        ptrs = self._cta_lists(h, lib, int(nL.sum()))
        for sweep, lev in (("factor", self._fwd_levels), ("fwd", self._fwd_levels), ("bwd", bl)):
            if sweep == "factor" and self._cta_nofactor:
                out[sweep] = None
                continue
            nlev = int(lev.max().item()) + 1
            o, lp = level_sort_dev(n, nlev, lev)
            order = np.ascontiguousarray(o[:n].cpu().numpy(), dtype=np.int32)
            lptr = np.ascontiguousarray(lp[:nlev + 1].cpu().numpy(), dtype=np.int32)
            kind = {"factor": 0, "fwd": 1, "bwd": 2}[sweep]
            sizes = (ctypes.c_int64 * 3)()
            args = [kind, n, _hp(rs), _hp(col), _hp(dg), _hp(order), _hp(lptr), nlev,
                    *ptrs, int(self.milu)]
            if lib.jv_cta_program_host(*args, None, None, sizes) != 0:
                out[sweep] = None          # too large for the single-CTA path
                continue
            total, maxblk, maxstage = (int(v) for v in sizes)
            if total > self.CTA_MAX_PROGRAM or 3 * 4 * maxblk > 200 * 1024:
                out[sweep] = None          # a level block cannot fit shared memory
                continue
            prog = np.empty(max(total, 4), dtype=np.int32)
            lbase = np.empty(nlev + 1, dtype=np.int32)
            _lib.call("jv_cta_program_host", *args, _hp(prog), _hp(lbase), sizes)
            # deepest pipeline that fits, values resident in shared memory first
            fit = [(res, rb) for res in (1, 0) for rb in self.CTA_RINGS
                   if lib.jv_cta_smem(kind, n, nnz, nlev, maxblk, maxstage, res, rb) >= 0]
            if not fit:
                out[sweep] = None
                continue
            resident, rb = fit[0]
            up = lambda a: t.from_numpy(a).to("cuda")
            out[sweep] = dict(kind=kind, prog=up(prog), lbase=up(lbase), nlev=nlev, maxblk=maxblk,
                              maxstage=maxstage, resident=resident, rb=rb,
                              maxrows=int(np.diff(lptr).max()) if nlev else 0)
        return out

    def _cta_lists(self, h, lib, nl):
        """Host copies (lstart, off, otgt, oq, ok) of the update lists."""
        info = (ctypes.c_int64 * 4)()
        _lib.call("jv_cta_plan_export", h, None, None, None, None, None, info)
        nops = int(info[1])
        if 2 * nops > self.CTA_MAX_PROGRAM:
            nops, nl = 0, 0     # the factor program would not fit: lists not needed
        lstart = np.empty(self.n + 1, np.int32)
        off = np.empty(nl + 1, np.int64)
        otgt = np.empty(max(nops, 1), np.int32)
        oq = np.empty(max(nops, 1), np.int32)
        ok = np.zeros(max(nops, 1), np.int8)
        if nl or nops:
            _lib.call("jv_cta_plan_export", h, _hp(lstart), _hp(off), _hp(otgt), _hp(oq), _hp(ok),
                      info)
        else:
            self._cta_nofactor = True
        self._cta_keep = (lstart, off, otgt, oq, ok)
        return [_hp(lstart), _hp(off), _hp(otgt), _hp(oq), _hp(ok)]

    def cta_ok(self, sweep):
        return self.cta_programs().get(sweep) is not None

    def _cta_run(self, sweep, inp=None, out=None):
        g = self.cta_programs()[sweep]
        _lib.call("jv_cta_run", g["kind"], self.n, self.nnz, g["nlev"], ptr(g["prog"]),
                  ptr(g["lbase"]), g["maxblk"], g["maxstage"], g["resident"], g["rb"], g["maxrows"],
                  ptr(self.val),
                  ptr(self.norms), self.tau, int(self.milu), ptr(inp), ptr(out), ptr(self.err),
                  stream())

    def _factor_cta(self, norms, reset=True):
        if norms and self.tau > 0:
            self.compute_norms()
        if reset:
            _lib.call("jv_reset_row", ptr(self.err), stream())
        self._cta_run("factor")

    def _solve_cta(self, which, b, out):
        self._cta_run("fwd" if which == 0 else "bwd", b, out)

    # small systems: one sweep in one thread block, all in shared memory ---
    def _level_lists(self, which):
        """(rows in level order (device int32), level bounds (numpy), depth)
        of one sweep's DAG, from its schedule."""
        sched = self.fwd_schedule() if which == 0 else self.bwd_schedule()
        nclass = len(sched.steps) if hasattr(sched, "steps") else 2
        order = sched.order
        lev = (sched.keys[order.long()] // nclass).cpu().numpy()
        nlev = int(lev.max()) + 1 if lev.size else 0
        return order, np.searchsorted(lev, np.arange(nlev + 1)), nlev

    def _small_plan(self, which):
        """Arguments of jv_solve_small for one direction, or None when the
        sweep does not fit one thread block's shared memory (cached)."""
        cache = self.__dict__.setdefault("_small", {})
        if which not in cache:
            t = torch()
            lib = _lib.load()
            plan = None
            if 0 < self.n <= (1 << 15):
                n = self.n
                rs, dg = self.row_start[:n + 1].long(), self.diag_pos[:n].long()
                cnt = (dg - rs[:n]) if which == 0 else (rs[1:] - dg - 1)
                nent = int(cnt.sum().item())
                order, lptr, nlev = self._level_lists(which)
                if lib.jv_solve_small_bytes(which, n, nlev, nent) <= lib.jv_solve_small_max():
                    estart = t.zeros(n + 1, dtype=t.int32, device="cuda")
                    estart[1:] = t.cumsum(cnt, 0).to(t.int32)
                    width = int(np.diff(lptr).max()) if nlev else 0
                    plan = (order.contiguous(), i32(lptr), nlev, estart, nent, width)
            cache[which] = plan
        return cache[which]

    def _solve_small(self, which, b, out):
        order, lptr, nlev, estart, nent, width = self._small_plan(which)
        _lib.call("jv_solve_small", which, self.n, ptr(self.row_start), ptr(self.col), ptr(self.val),
                  ptr(self.diag_pos), ptr(order), ptr(lptr), nlev, ptr(estart), nent, width, ptr(b),
                  ptr(out), stream())

    # streamed drop-in factorization: host values in, factors out -------
    STREAM_CHUNKS = 8

    STREAM_ENDS = 2       # small chunks at each end (pipeline fill and drain)

    def _chunks(self, k):
        """Row bounds of k chunks balanced by stored entries, plus
        STREAM_ENDS chunks of a quarter size at both ends, so the pipeline
        fills and drains quickly (cached)."""
        key = ("chunks", k, self.STREAM_ENDS)
        if getattr(self, "_chunk_cache", None) is None or self._chunk_cache[0] != key:
            rs = self._host_pattern()[0].astype(np.int64)
            e = 1.0 / (4 * k)
            ends = [e * i for i in range(1, self.STREAM_ENDS + 1)]
            inner = np.linspace(ends[-1] if ends else 0.0, 1.0 - (ends[-1] if ends else 0.0),
                                k + 1)
            fr = np.unique(np.concatenate([[0.0], ends, inner, [1.0 - x for x in ends], [1.0]]))
            tgt = fr * self.nnz
            b = np.unique(np.searchsorted(rs, tgt, side="left").clip(0, self.n))
            b[0], b[-1] = 0, self.n
            self._chunk_cache = (key, b, rs)
        return self._chunk_cache[1], self._chunk_cache[2]

    def factor_streamed(self, host_val):
        """factor_serial with host values (a page-locked float64 array, read
        and overwritten in place): the rows are cut into chunks in level
        order; chunk c's upload, chunk c-1's factorization (sync-free kernel
        over those rows, earlier rows final) and chunk c-2's download run
        concurrently on three streams, so the host link in both directions
        overlaps the device work.  Returns the smallest zero-pivot row or -1;
        rows after it get their input values back (the reference stops
        there)."""
        t = torch()
        main = t.cuda.current_stream()
        if getattr(self, "_xfer", None) is None:
            self._xfer = (t.cuda.Stream(), t.cuda.Stream())
            self._vbak = None
        s_in, s_out = self._xfer
        if self._vbak is None or self._vbak.numel() < self.nnz:
            self._vbak = empty_f64(self.nnz)
        bounds, rs = self._chunks(self.STREAM_CHUNKS)
        hp = host_val.ctypes.data
        dp = self.val.data_ptr()
        s_in.wait_stream(main)
        _lib.call("jv_reset_row", ptr(self.err), stream())
        done_in, done_f = [], []
        for c in range(bounds.size - 1):
            lo, hi = int(bounds[c]), int(bounds[c + 1])
            p0, p1 = int(rs[lo]), int(rs[hi])
            if p1 > p0:
                _lib.call("jv_memcpy_async", ctypes.c_void_p(dp + 8 * p0),
                          ctypes.c_void_p(hp + 8 * p0), 8 * (p1 - p0), 0,
                          ctypes.c_void_p(s_in.cuda_stream))
            e = t.cuda.Event()
            e.record(s_in)
            done_in.append(e)
        for c in range(bounds.size - 1):
            lo, hi = int(bounds[c]), int(bounds[c + 1])
            p0, p1 = int(rs[lo]), int(rs[hi])
            main.wait_event(done_in[c])
            self._vbak[p0:p1].copy_(self.val[p0:p1])
            if self.tau > 0 and hi > lo:
                _lib.call("jv_row_norms", hi - lo, ctypes.c_void_p(self.row_start.data_ptr() + 4 * lo),
                          ptr(self.val), self.tau, ctypes.c_void_p(self.norms.data_ptr() + 8 * lo),
                          stream())
            if hi > lo:
                self._factor_tickets(lo, hi, lo, False, reset=False)
            e = t.cuda.Event()
            e.record(main)
            done_f.append(e)
            s_out.wait_event(e)
            if p1 > p0:
                _lib.call("jv_memcpy_async", ctypes.c_void_p(hp + 8 * p0),
                          ctypes.c_void_p(dp + 8 * p0), 8 * (p1 - p0), 1,
                          ctypes.c_void_p(s_out.cuda_stream))
        main.wait_stream(s_out)
        self.values_changed()
        bad = read_row_slot(self.err)
        check_hang()
        if bad >= 0:
            p = int(rs[bad + 1])
            if p < self.nnz:
                _lib.call("jv_memcpy_async", ctypes.c_void_p(hp + 8 * p),
                          ctypes.c_void_p(self._vbak.data_ptr() + 8 * p), 8 * (self.nnz - p), 1,
                          stream())
                self.val[p:self.nnz].copy_(self._vbak[p:self.nnz])
            sync()
        return bad

    def factor(self, lo=0, hi=None, ready_below=0):
        """Factor and return the smallest zero-pivot row (or -1)."""
        self.factor_async(lo, hi, ready_below)
        bad = read_row_slot(self.err)
        check_hang()
        return bad

    def first_zero_diag(self):
        slot = reset_row_slot()
        _lib.call("jv_check_zero_diag", self.n, ptr(self.val), ptr(self.diag_pos), ptr(slot),
                  stream())
        return read_row_slot(slot)

    def solve_async(self, which, b, out):
        rp = self._region_for("fwd" if which == 0 else "bwd")
        if rp is CTA:
            self._solve_cta(which, b, out)
            return out
        if rp is SMALL:
            self._solve_small(which, b, out)
            return out
        if rp is not None:
            # the backward sweep's value pack depends only on the factors:
            # refresh it on a side stream while the forward region kernel
            # runs, when that kernel leaves most SMs idle (one CTA per
            # region; with more regions the pack slows the sweep down more
            # than it saves: c4 fwd 0.95 -> 1.14 ms)
            nxt = None
            if self._sms is None:
                t = torch()
                self._sms = t.cuda.get_device_properties(t.cuda.current_device()).multi_processor_count
            if which == 0 and 2 * rp["nreg"] <= self._sms:
                nxt = (self._rchoice.get(("bwd", False)) if self.region_mode == "auto"
                       else self.region_stream("bwd"))
            ev = []
            hook = None
            if nxt is not None and "pver" in nxt and nxt["pver"] != self._vver:   # (a region plan)
                hook = lambda: ev.append(self._side_pack(nxt))
            self._region_run(rp, 1 + which, b, out, self.sbox, hook)
            if ev:
                torch().cuda.current_stream().wait_event(ev[0])
            return out
        self._solve_tickets(which, b, out)
        return out

    def _solve_tickets(self, which, b, out):
        sched = self.fwd_schedule() if which == 0 else self.bwd_schedule()
        _lib.call("jv_solve", which, self.n, ptr(self.row_start), ptr(self.col), ptr(self.val),
                  ptr(self.diag_pos), ptr(sched.order), ptr(sched.batch_ptr), sched.nbatch,
                  ptr(b), ptr(out), ptr(self.sbox.buf), self.sbox.next_epoch(),
                  ctypes.c_void_p(self.ticket.data_ptr() + 8), stream())

    # the paper's CSR-LS baseline on the GPU ----------------------------
    def _csrls_graph(self, which):
        """CUDA graph of one level-synchronous sweep (one launch per level)
        over fixed in/out buffers; built once per pattern and direction."""
        if which in self._csrls:
            return self._csrls[which]
        t = torch()
        sched = self.fwd_schedule() if which == 0 else self.bwd_schedule()
        nclass = len(sched.steps) if hasattr(sched, "steps") else 2
        order = sched.order
        keys = sched.keys[order.long()] // nclass
        lev = keys.cpu().numpy()
        nlev = int(lev.max()) + 1 if lev.size else 0
        ptr_ = np.searchsorted(lev, np.arange(nlev + 1))
        bin_ = t.zeros(self.n, dtype=t.float64, device="cuda")
        bout = t.zeros(self.n, dtype=t.float64, device="cuda")
        args = (ptr(self.row_start), ptr(self.col), ptr(self.val), ptr(self.diag_pos), ptr(order))
        s = t.cuda.Stream()
        s.wait_stream(t.cuda.current_stream())
        with t.cuda.stream(s):   # warm-up outside capture
            for L in range(nlev):
                _lib.load().jv_solve_level(which, *args, int(ptr_[L]), int(ptr_[L + 1]), ptr(bin_),
                                           ptr(bout), stream())
        t.cuda.current_stream().wait_stream(s)
        g = t.cuda.CUDAGraph()
        with t.cuda.graph(g):
            for L in range(nlev):
                _lib.load().jv_solve_level(which, *args, int(ptr_[L]), int(ptr_[L + 1]), ptr(bin_),
                                           ptr(bout), stream())
        self._csrls[which] = (g, bin_, bout, nlev)
        return self._csrls[which]

    def solve_csrls_async(self, which, b, out):
        """Level-synchronous sweep (the paper's CSR-LS baseline): bitwise the
        same result as solve_async."""
        g, bin_, bout, nlev = self._csrls_graph(which)
        bin_.copy_(b[:self.n])
        g.replay()
        _lib.launch_counts["jv_solve_level"] = _lib.launch_counts.get("jv_solve_level", 0) + nlev
        out[:self.n].copy_(bout)
        return out

    def host_val(self):
        return host_f64(self.val, self.nnz)
