"""Dependency levels, the two-stage (upper block / lower tail) partition and
the RCM base ordering — the reference ordering.py API
(/root/reference/pkg/src/ilukit/ordering.py) with the level sets and the
partition rule computed on the GPU (libjv: jv_levels, jv_level_sort,
jv_partition), bit-exact with the reference.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from . import device as dv
from .csr import Permutation, SparsityPattern, symmetrize_pattern
from .errors import ConfigurationError

__all__ = [
    "LOWER_A",
    "LOWER_A_PLUS_AT",
    "BACKWARD_UPPER",
    "LevelSchedule",
    "PartitionConfig",
    "StagePartition",
    "compute_levels",
    "compute_levels_backward",
    "partition_stages",
    "build_level_permutation",
    "contiguous_partition",
    "rcm_order",
    "level_stats",
]

LOWER_A = "lower_A"
LOWER_A_PLUS_AT = "lower_AplusAT"
BACKWARD_UPPER = "backward_upper"


@dataclass
class LevelSchedule:
    """Row -> level plus per-level row lists, level-ascending (ordering.py:37-51)."""

    level_of: np.ndarray
    levels: list
    source_pattern_kind: str

    @property
    def num_levels(self) -> int:
        return len(self.levels)

    @property
    def n(self) -> int:
        return self.level_of.size


@dataclass
class PartitionConfig:
    min_level_rows: int = 16
    density_factor: float = 4.0
    suffix_only: bool = True

    def validate(self) -> None:
        if self.min_level_rows < 1:
            raise ConfigurationError("min_level_rows must be >= 1")
        if not self.density_factor > 0:
            raise ConfigurationError("density_factor must be positive")


@dataclass
class StagePartition:
    """Levels kept for the scheduled stage plus the rows moved to the end."""

    upper_levels: list
    lower_rows: np.ndarray
    cut_level: int
    config: PartitionConfig = field(default_factory=PartitionConfig)
    levels_kind: str = LOWER_A_PLUS_AT

    @property
    def n_upper(self) -> int:
        return sum(len(l) for l in self.upper_levels)

    @property
    def n(self) -> int:
        return self.n_upper + len(self.lower_rows)


def _schedule_from_device(level_of_d, nlev, n, kind) -> LevelSchedule:
    order_d, level_ptr_d = dv.level_sort_dev(n, nlev, level_of_d)
    level_of = dv.host_i64(level_of_d, n)
    order = dv.host_i64(order_d, n)
    level_ptr = dv.host_i64(level_ptr_d, nlev + 1)
    levels = [order[level_ptr[i]:level_ptr[i + 1]] for i in range(nlev)]
    return LevelSchedule(level_of, levels, kind)


def compute_levels(lower: SparsityPattern, kind: str = LOWER_A) -> LevelSchedule:
    """Longest-path levels of a strictly lower-triangular dependency pattern
    (reference ordering.py:97-104 -> _kernels.py:37-48)."""
    if lower.n == 0:
        return LevelSchedule(np.zeros(0, dtype=np.int64), [], kind)
    d = dv.DevCsr.from_host(lower.n, lower.row_start, lower.col)
    level_of_d, nlev = dv.levels_dev(d, backward=False)
    return _schedule_from_device(level_of_d, nlev, lower.n, kind)


def compute_levels_backward(pattern: SparsityPattern) -> LevelSchedule:
    """Levels of the backward sweep: row i waits on j > i
    (reference ordering.py:107-116 -> _kernels.py:51-62)."""
    if pattern.n == 0:
        return LevelSchedule(np.zeros(0, dtype=np.int64), [], BACKWARD_UPPER)
    d = dv.DevCsr.from_host(pattern.n, pattern.row_start, pattern.col)
    level_of_d, nlev = dv.levels_dev(d, backward=True)
    return _schedule_from_device(level_of_d, nlev, pattern.n, BACKWARD_UPPER)


def _partition_rule_host(levels, row_nnz, config):
    """Reference rule evaluated with numpy means; used only when row_nnz is
    not integral (real row counts always take the device path)."""
    mean_nnz = row_nnz.mean() if row_nnz.size else 0.0
    ok = [
        len(rows) >= config.min_level_rows
        and (row_nnz[rows].mean() if len(rows) else 0.0) <= config.density_factor * mean_nnz
        for rows in levels
    ]
    cut = len(levels)
    if config.suffix_only:
        while cut > 0 and not ok[cut - 1]:
            cut -= 1
    else:
        for i, good in enumerate(ok):
            if not good:
                cut = i
                break
    return cut


def partition_stages(
    schedule: LevelSchedule,
    row_nnz: np.ndarray,
    config: PartitionConfig | None = None,
) -> StagePartition:
    """Split levels into the scheduled (upper) stage and a trailing excluded
    suffix (reference ordering.py:119-159): a level is acceptable when it has
    >= min_level_rows rows and mean row density <= density_factor x matrix
    mean; only a failing suffix is cut (first failure when suffix_only is
    off)."""
    config = config or PartitionConfig()
    config.validate()
    row_nnz = np.asarray(row_nnz)
    levels = schedule.levels
    nlev = len(levels)
    integral = (
        row_nnz.size > 0
        and np.all(np.isfinite(row_nnz))
        and np.all(np.asarray(row_nnz, dtype=np.float64) == np.round(row_nnz))
        and np.abs(row_nnz).max() < 2**31
    )
    if nlev == 0:
        cut = 0
    elif integral and row_nnz.size == schedule.n:
        order = np.concatenate(levels).astype(np.int64)
        level_ptr = np.zeros(nlev + 1, dtype=np.int64)
        np.cumsum([len(l) for l in levels], out=level_ptr[1:])
        cut_h = ctypes.c_int32(0)
        nup_h = ctypes.c_int32(0)
        # keep the device tensors referenced until the call has been issued
        lp_d = dv.i32(level_ptr)
        order_d = dv.i32(order)
        nnz_d = dv.i32(np.asarray(row_nnz, dtype=np.int64))
        _lib.call(
            "jv_partition", schedule.n, nlev, dv.ptr(lp_d), dv.ptr(order_d), dv.ptr(nnz_d),
            int(config.min_level_rows), float(config.density_factor),
            int(bool(config.suffix_only)), ctypes.byref(cut_h), ctypes.byref(nup_h), dv.stream(),
        )
        cut = int(cut_h.value)
    else:
        cut = _partition_rule_host(levels, row_nnz, config)
    upper = [np.array(rows, copy=True) for rows in levels[:cut]]
    lower = (
        np.concatenate([levels[i] for i in range(cut, nlev)])
        if cut < nlev
        else np.zeros(0, dtype=np.int64)
    )
    return StagePartition(upper, lower, cut, config, schedule.source_pattern_kind)


def build_level_permutation(partition: StagePartition) -> Permutation:
    """new -> old ordering: upper levels in order, then the excluded rows."""
    pieces = list(partition.upper_levels) + [partition.lower_rows]
    perm = np.concatenate(pieces) if pieces else np.zeros(0, dtype=np.int64)
    return Permutation(perm.astype(np.int64))


def contiguous_partition(partition: StagePartition) -> StagePartition:
    """The same partition re-indexed after its own level permutation."""
    sizes = [len(l) for l in partition.upper_levels]
    bounds = np.zeros(len(sizes) + 1, dtype=np.int64)
    np.cumsum(sizes, out=bounds[1:])
    upper = [np.arange(bounds[i], bounds[i + 1]) for i in range(len(sizes))]
    lower = np.arange(partition.n_upper, partition.n, dtype=np.int64)
    return StagePartition(upper, lower, partition.cut_level, partition.config,
                          partition.levels_kind)


def level_stats(schedule: LevelSchedule) -> dict:
    """Level count and row-count extremes; median = lower middle element."""
    sizes = sorted(len(l) for l in schedule.levels)
    if not sizes:
        return {"num_levels": 0, "min_rows": 0, "max_rows": 0, "median_rows": 0}
    return {
        "num_levels": len(sizes),
        "min_rows": sizes[0],
        "max_rows": sizes[-1],
        "median_rows": sizes[(len(sizes) - 1) // 2],
    }


def rcm_order(pattern: SparsityPattern) -> Permutation:
    """Reverse Cuthill-McKee on the symmetrized pattern (reference
    ordering.py:199-266): pseudo-peripheral roots from minimum-degree
    vertices, neighbours by (degree, index), order reversed.  On the device
    (jv_rcm_device: level-synchronous Cuthill-McKee, bit-exact); a graph with
    more than 64 components of two or more vertices goes to libjv's host C++
    (jv_rcm_host, same result), where per-component launches would dominate."""
    n = pattern.n
    if n == 0:
        return Permutation(np.zeros(0, dtype=np.int64))
    sym = symmetrize_pattern(pattern)
    rs = np.ascontiguousarray(sym.row_start, dtype=np.int32)
    col = np.ascontiguousarray(sym.col, dtype=np.int32)
    d = dv.DevCsr.from_host(n, rs, col)
    perm_d = dv.empty_i32(n)
    ncomp = ctypes.c_int32(0)
    rc = _lib.load().jv_rcm_device(n, dv.ptr(d.row_start), dv.ptr(d.col), dv.ptr(perm_d),
                                   RCM_DEVICE_MAX_COMPONENTS, ctypes.byref(ncomp), dv.stream())
    if rc == 0:
        return Permutation(dv.host_i64(perm_d, n))
    if rc != 1:
        raise RuntimeError("jv_rcm_device failed: " + _lib.load().jv_last_error().decode())
    perm = np.empty(n, dtype=np.int32)
    _lib.call("jv_rcm_host", n, rs.ctypes.data_as(ctypes.c_void_p),
              col.ctypes.data_as(ctypes.c_void_p), perm.ctypes.data_as(ctypes.c_void_p))
    return Permutation(perm.astype(np.int64))


RCM_DEVICE_MAX_COMPONENTS = 64


def rcm_order_host(pattern: SparsityPattern) -> Permutation:
    """The same ordering computed by libjv's host C++ (jv_rcm_host)."""
    n = pattern.n
    if n == 0:
        return Permutation(np.zeros(0, dtype=np.int64))
    sym = symmetrize_pattern(pattern)
    rs = np.ascontiguousarray(sym.row_start, dtype=np.int32)
    col = np.ascontiguousarray(sym.col, dtype=np.int32)
    perm = np.empty(n, dtype=np.int32)
    _lib.call("jv_rcm_host", n, rs.ctypes.data_as(ctypes.c_void_p),
              col.ctypes.data_as(ctypes.c_void_p), perm.ctypes.data_as(ctypes.c_void_p))
    return Permutation(perm.astype(np.int64))
