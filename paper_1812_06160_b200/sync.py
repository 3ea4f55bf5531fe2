"""Point-to-point schedule objects — the reference sync.py API
(/root/reference/pkg/src/ilukit/sync.py).

On the CPU the reference deals rows round-robin to worker threads and
prunes each row's waits to a minimal set (build_waits_kernel,
_kernels.py:94-151).  The GPU kernels need neither: every row awaits its own
dependencies through mailbox packets.  These objects are kept because they
are part of the API (solve setups, factor_parallel_upper); their `order`
(the rows covered) is what the GPU path uses.  Waits are the full structural
dependency lists (a superset of the reference's pruned lists, equally
valid); levels are computed on the GPU.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import device as dv
from .csr import SparsityPattern
from .errors import ConfigurationError
from .ordering import StagePartition

__all__ = ["SyncSchedule", "build_sync_schedule", "build_triangle_schedule"]


@dataclass
class SyncSchedule:
    """Worker assignment, per-worker program order and waits (sync.py:29-56)."""

    nthreads: int
    owner: np.ndarray
    pos: np.ndarray
    prog_ptr: np.ndarray
    prog_rows: np.ndarray
    wait_ptr: np.ndarray
    wait_rows: np.ndarray
    order: np.ndarray

    @property
    def flag_size(self) -> int:
        return self.wait_ptr.size - 1

    @property
    def total_waits(self) -> int:
        return int(self.wait_rows.size)

    def waits_of(self, r: int) -> np.ndarray:
        return self.wait_rows[self.wait_ptr[r]:self.wait_ptr[r + 1]]


def _triangle_deps(pattern: SparsityPattern, which: str, row_limit=None):
    owner = np.repeat(np.arange(pattern.n, dtype=np.int64), np.diff(pattern.row_start))
    if which == "forward":
        keep = pattern.col < owner
    elif which == "backward":
        keep = pattern.col > owner
    else:
        raise ValueError(f"unknown triangle {which!r}")
    if row_limit is not None:
        keep &= owner < row_limit
    dep_ptr = np.zeros(pattern.n + 1, dtype=np.int64)
    np.cumsum(np.bincount(owner[keep], minlength=pattern.n), out=dep_ptr[1:])
    return dep_ptr, pattern.col[keep].astype(np.int64)


def _make_schedule(levels, dep_ptr, dep_col, n, nthreads) -> SyncSchedule:
    if nthreads < 1:
        raise ConfigurationError("worker count must be >= 1")
    order = np.concatenate(levels).astype(np.int64) if levels else np.zeros(0, dtype=np.int64)
    covered = np.zeros(n, dtype=bool)
    covered[order] = True
    if dep_col.size and not covered[dep_col].all():
        raise ConfigurationError("dependency target outside the scheduled rows")
    k = np.arange(order.size, dtype=np.int64)
    owner = np.zeros(n, dtype=np.int64)
    pos = np.zeros(n, dtype=np.int64)
    owner[order] = k % nthreads
    pos[order] = k // nthreads
    prog_ptr = np.zeros(nthreads + 1, dtype=np.int64)
    np.cumsum(np.bincount(k % nthreads, minlength=nthreads), out=prog_ptr[1:])
    prog_rows = order[np.argsort(k % nthreads, kind="stable")]
    # full structural waits, rows outside `order` get none
    counts = np.diff(dep_ptr) * covered
    wait_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=wait_ptr[1:])
    sel = np.repeat(covered, np.diff(dep_ptr))
    return SyncSchedule(nthreads, owner, pos, prog_ptr, prog_rows, wait_ptr, dep_col[sel], order)


def build_sync_schedule(
    partition: StagePartition, pattern: SparsityPattern, nthreads: int
) -> SyncSchedule:
    """Schedule of the upper-stage rows (sync.py:119-149)."""
    if partition.n_upper < pattern.n:
        from .lower import _check_level_order

        _check_level_order(partition, pattern.n)
    dep_ptr, dep_col = _triangle_deps(pattern, "forward", partition.n_upper)
    return _make_schedule(list(partition.upper_levels), dep_ptr, dep_col, pattern.n, nthreads)


def build_triangle_schedule(
    pattern: SparsityPattern, nthreads: int, which: str
) -> SyncSchedule:
    """Schedule over all rows for one sweep direction (sync.py:152-168);
    levels from the GPU level kernels."""
    dep_ptr, dep_col = _triangle_deps(pattern, which)
    if pattern.n == 0:
        return _make_schedule([], dep_ptr, dep_col, 0, nthreads)
    d = dv.DevCsr.from_host(pattern.n, pattern.row_start, pattern.col)
    level_of_d, nlev = dv.levels_dev(d, backward=(which == "backward"))
    order_d, level_ptr_d = dv.level_sort_dev(pattern.n, nlev, level_of_d)
    order = dv.host_i64(order_d, pattern.n)
    lp = dv.host_i64(level_ptr_d, nlev + 1)
    levels = [order[lp[i]:lp[i + 1]] for i in range(nlev)]
    return _make_schedule(levels, dep_ptr, dep_col, pattern.n, nthreads)
