"""Multi-GPU paths: the two parts of the hot path that shard.

* Row-partitioned spmv.  Contiguous row blocks balanced by nnz, x
  partitioned the same way, ONE halo exchange per product: each rank packs
  the x entries its neighbours read (jv_gather), the blocks travel as grouped
  point-to-point sends/receives (torch.distributed -> NCCL over NVLink), and
  the interior rows (no remote column) are multiplied while the exchange is
  in flight; the boundary rows follow once it lands (jv_spmv_rows with a row
  map, so both halves write straight into y).  The local x lives in the
  middle of an extended vector [ghosts of lower ranks | own block | ghosts of
  higher ranks]: owner blocks are contiguous and ascending, so the remapped
  column indices keep every row's column order and each row's sum is the
  same sequence of roundings as the single-GPU product (csr.py:251-260) —
  bitwise equal.
* Batches of independent systems (config 5): rank p takes a contiguous
  block of the batch and factors / solves it alone (one block-diagonal
  matrix per rank); no collective on the hot path.

Factorization and stri of ONE matrix are replicas only (one GPU per
matrix).

The communication is plain torch.distributed (NCCL for CUDA tensors, gloo
for the CPU tests); the compute goes through an `ops` object — libjv
kernels on the GPU (DeviceOps), a numpy stand-in in the gloo tests.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

__all__ = ["row_partition", "HaloPlan", "plan_halo", "DistSpmv", "DeviceOps", "shard_range",
           "BatchShard"]


def row_partition(row_start, parts: int) -> np.ndarray:
    """Row bounds [parts+1] of contiguous blocks with ~equal nonzeros."""
    rs = np.asarray(row_start, dtype=np.int64)
    n = rs.size - 1
    nnz = int(rs[-1])
    targets = (np.arange(1, parts, dtype=np.int64) * nnz) // parts
    cuts = np.searchsorted(rs, targets, side="left")
    bounds = np.concatenate([[0], np.clip(cuts, 0, n), [n]]).astype(np.int64)
    return np.maximum.accumulate(bounds)


def shard_range(count: int, rank: int, world: int) -> range:
    """Contiguous block of a batch of `count` independent systems."""
    lo = (count * rank) // world
    hi = (count * (rank + 1)) // world
    return range(lo, hi)


@dataclass
class HaloPlan:
    rank: int
    world: int
    bounds: np.ndarray          # row bounds of every rank
    lo: int
    hi: int
    n_below: int                # ghosts owned by lower ranks (ext prefix)
    n_above: int                # ghosts owned by higher ranks (ext suffix)
    recv: list                  # (peer, ext offset, count), ascending peer
    send: list                  # (peer, local indices into the own block)
    rs: np.ndarray              # local CSR over ext columns
    col: np.ndarray
    val: np.ndarray
    interior: np.ndarray        # local rows with only own-block columns
    boundary: np.ndarray        # the others
    halo_bytes: int = 0         # x bytes received per product
    stats: dict = field(default_factory=dict)

    @property
    def n_local(self):
        return self.hi - self.lo

    @property
    def n_ext(self):
        return self.n_below + self.n_local + self.n_above


def _exchange_needs(needs, rank, world, group):
    """needs[q] = global columns this rank reads from q; returns what every
    peer reads from this rank (setup only: all_gather of the index lists)."""
    import torch.distributed as dist

    everyone = [None] * world
    dist.all_gather_object(everyone, needs, group=group)
    return {q: everyone[q][rank] for q in range(world) if q != rank and rank in everyone[q]}


def _needs(lcol, bounds, rank):
    owner = np.searchsorted(bounds, lcol, side="right") - 1
    remote = owner != rank
    return {int(q): np.unique(lcol[owner == q]) for q in np.unique(owner[remote])}, remote


def plan_halo(row_start, col, val, bounds, rank, world, group=None, peers_need=None) -> HaloPlan:
    """Partition plan of rank `rank` for the matrix (this rank needs only its
    own rows; the peers' needs arrive through one all_gather unless given)."""
    rs = np.asarray(row_start, dtype=np.int64)
    lo, hi = int(bounds[rank]), int(bounds[rank + 1])
    a, b = int(rs[lo]), int(rs[hi])
    lcol = np.asarray(col[a:b], dtype=np.int64)
    lval = np.asarray(val[a:b], dtype=np.float64)
    lrs = rs[lo:hi + 1] - a
    needs, remote = _needs(lcol, bounds, rank)
    if peers_need is None:
        peers_need = _exchange_needs(needs, rank, world, group) if world > 1 else {}
    below = [q for q in sorted(needs) if q < rank]
    above = [q for q in sorted(needs) if q > rank]
    ghosts_lo = np.concatenate([needs[q] for q in below]) if below else np.zeros(0, np.int64)
    ghosts_hi = np.concatenate([needs[q] for q in above]) if above else np.zeros(0, np.int64)
    n_below, n_local = ghosts_lo.size, hi - lo
    # ext index: monotone in the global column
    ext = np.empty_like(lcol)
    loc = ~remote
    ext[loc] = lcol[loc] - lo + n_below
    m_lo = remote & (lcol < lo)
    m_hi = remote & (lcol >= hi)
    ext[m_lo] = np.searchsorted(ghosts_lo, lcol[m_lo])
    ext[m_hi] = n_below + n_local + np.searchsorted(ghosts_hi, lcol[m_hi])
    recv, off = [], 0
    for q in below:
        recv.append((q, off, needs[q].size))
        off += needs[q].size
    off = n_below + n_local
    for q in above:
        recv.append((q, off, needs[q].size))
        off += needs[q].size
    send = [(q, np.asarray(peers_need[q], dtype=np.int64) - lo) for q in sorted(peers_need)]
    row_remote = np.zeros(n_local, dtype=bool)
    if remote.any():
        rows = np.repeat(np.arange(n_local), np.diff(lrs))
        row_remote[np.unique(rows[remote])] = True
    plan = HaloPlan(rank, world, np.asarray(bounds, dtype=np.int64), lo, hi, n_below,
                    ghosts_hi.size, recv, send, lrs, ext, lval,
                    np.flatnonzero(~row_remote), np.flatnonzero(row_remote))
    plan.halo_bytes = 8 * (ghosts_lo.size + ghosts_hi.size)
    plan.stats = {"peers": len(recv), "ghosts": int(ghosts_lo.size + ghosts_hi.size),
                  "boundary_rows": int(plan.boundary.size), "nnz": int(lrs[-1])}
    return plan


def plan_halo_all(row_start, col, bounds_or_parts, val=None):
    """Every rank's plan in one process (tests / single-process emulation of
    the exchange): the needs of all ranks are computed here directly."""
    rs = np.asarray(row_start, dtype=np.int64)
    col = np.asarray(col)
    val = np.zeros(col.size) if val is None else np.asarray(val)
    bounds = (row_partition(rs, bounds_or_parts) if np.isscalar(bounds_or_parts)
              else np.asarray(bounds_or_parts, dtype=np.int64))
    world = bounds.size - 1
    needs = [_needs(np.asarray(col[rs[bounds[p]]:rs[bounds[p + 1]]], dtype=np.int64), bounds, p)[0]
             for p in range(world)]
    plans = []
    for p in range(world):
        peers = {q: needs[q][p] for q in range(world) if q != p and p in needs[q]}
        plans.append(plan_halo(rs, col, val, bounds, p, world, peers_need=peers))
    return plans


def _sub_csr(rs, col, val, rows):
    """CSR of the given local rows (kept in order)."""
    lens = np.diff(rs)[rows]
    srs = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    total = int(srs[-1])
    take = np.repeat(rs[rows] - srs[:-1], lens) + np.arange(total, dtype=np.int64)
    return srs, col[take], val[take]


class DeviceOps:
    """libjv kernels on CUDA tensors (the product path)."""

    def __init__(self):
        from . import device as dv
        self.dv = dv

    def tensor_i32(self, a):
        return self.dv.i32(a) if len(a) else self.dv.empty_i32(1)

    def tensor_f64(self, a):
        return self.dv.f64(a) if len(a) else self.dv.empty_f64(1)

    def empty_f64(self, n):
        return self.dv.empty_f64(max(int(n), 1))

    def csr(self, rs, col, val):
        d = self.dv.DevCsr.from_host(rs.size - 1, rs, col, val)
        d.tile_rows()
        return d

    def gather(self, idx, n, src, dst):
        from . import _lib
        _lib.call("jv_gather", n, self.dv.ptr(idx), self.dv.ptr(src), self.dv.ptr(dst),
                  self.dv.stream())

    def spmv_rows(self, csr, x, y, row_map):
        from . import _lib
        dv = self.dv
        _lib.call("jv_spmv_rows", csr.n, csr.nnz, dv.ptr(csr.row_start), dv.ptr(csr.col),
                  dv.ptr(csr.val), dv.ptr(x), dv.ptr(y), dv.ptr(csr.tile_rows()),
                  dv.ptr(row_map), dv.stream())


class DistSpmv:
    """y_local = (A x)[lo:hi] with one halo exchange (see module doc)."""

    def __init__(self, plan: HaloPlan, ops=None, group=None):
        self.plan = plan
        self.ops = ops if ops is not None else DeviceOps()
        self.group = group
        o = self.ops
        self.x_ext = o.empty_f64(plan.n_ext)
        self.x_local = self.x_ext[plan.n_below:plan.n_below + plan.n_local]
        self.parts = []
        for rows in (plan.interior, plan.boundary):
            if rows.size == 0:
                self.parts.append(None)
                continue
            srs, scol, sval = _sub_csr(plan.rs, plan.col, plan.val, rows)
            self.parts.append((o.csr(srs, scol, sval), o.tensor_i32(rows)))
        self.send = [(q, o.tensor_i32(idx), idx.size, o.empty_f64(idx.size)) for q, idx in plan.send]
        import torch.distributed as dist
        if plan.world > 1 and dist.is_available() and dist.is_initialized():
            # NCCL requires the first collective on a communicator to include
            # every rank; a rank without halo peers would otherwise never
            # join it.  One tiny all-reduce at plan time initialises it.
            # (Without a process group: single-process emulation, tests.)
            probe = self.x_ext.new_zeros(1)
            dist.all_reduce(probe, group=group)

    def _post(self):
        import torch.distributed as dist
        self.pack()
        ops = []
        for q, idx, m, buf in self.send:
            ops.append(dist.P2POp(dist.isend, buf[:m], q, group=self.group))
        for q, off, m in self.plan.recv:
            ops.append(dist.P2POp(dist.irecv, self.x_ext[off:off + m], q, group=self.group))
        return dist.batch_isend_irecv(ops) if ops else []

    def pack(self):
        """Gather the entries every peer reads into the send buffers."""
        for q, idx, m, buf in self.send:
            self.ops.gather(idx, m, self.x_local, buf)

    def interior(self, y_local):
        if self.parts[0] is not None:
            csr, rmap = self.parts[0]
            self.ops.spmv_rows(csr, self.x_ext, y_local, rmap)

    def boundary(self, y_local):
        if self.parts[1] is not None:
            csr, rmap = self.parts[1]
            self.ops.spmv_rows(csr, self.x_ext, y_local, rmap)

    def __call__(self, x_local, y_local):
        """x_local: this rank's block of x (may be self.x_local itself, then
        no copy); y_local receives this rank's rows of A x."""
        if x_local.data_ptr() != self.x_local.data_ptr():
            self.x_local.copy_(x_local)
        works = self._post()
        self.interior(y_local)        # overlaps the exchange
        for w in works:
            w.wait()
        self.boundary(y_local)
        return y_local


class BatchShard:
    """Batch sharding of independent systems (config 5):
    rank p owns the contiguous block shard_range(count, p, world) of the
    batch, stacks it into one block-diagonal matrix (workloads.block_diagonal)
    and factors / solves it with no collective on the hot path; per-system
    results are cut back out of the level-permuted storage (the level
    permutation keeps every block's rows in their relative order) and,
    off the hot path, gathered as records on every rank."""

    def __init__(self, count: int, rank: int = 0, world: int = 1, first: int = 0):
        self.count, self.rank, self.world, self.first = count, rank, world, first
        self.seeds = [first + s for s in shard_range(count, rank, world)]
        self.sizes = []

    def assemble(self, make):
        """Block-diagonal matrix of this rank's systems (`make(seed)` -> CsrMatrix)."""
        from .workloads import block_diagonal
        mats = [make(sd) for sd in self.seeds]
        self.sizes = [m.n for m in mats]
        return block_diagonal(mats)

    def system_rows(self, perm):
        """{seed: rows of that system in the level-permuted order}."""
        perm = np.asarray(perm, dtype=np.int64)
        out, off = {}, 0
        for sd, m in zip(self.seeds, self.sizes):
            out[sd] = np.flatnonzero((perm >= off) & (perm < off + m))
            off += m
        return out

    @staticmethod
    def take_rows(row_start, val, rows):
        """The stored values of `rows` (in order), e.g. one system's factor."""
        rs = np.asarray(row_start, dtype=np.int64)
        lens = rs[rows + 1] - rs[rows]
        starts = np.concatenate([[0], np.cumsum(lens)])[:-1]
        idx = np.repeat(rs[rows] - starts, lens) + np.arange(int(lens.sum()))
        return np.asarray(val)[idx]

    def gather(self, records, group=None):
        """All ranks' {seed: record} merged on every rank (off the hot path)."""
        if self.world == 1:
            return dict(records)
        import torch.distributed as dist
        parts = [None] * self.world
        dist.all_gather_object(parts, dict(records), group=group)
        out = {}
        for p in parts:
            out.update(p)
        return out
