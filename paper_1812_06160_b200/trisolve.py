"""Sparse triangular solves (stri) over the combined L|U storage — the
reference trisolve.py API (/root/reference/pkg/src/ilukit/trisolve.py)
backed by the sync-free sm_100a kernels of jv_solve.

The reference's four paths (serial sweeps, CSR-LS barriers, pruned p2p,
two-stage) are bitwise identical by construction; on the GPU all of them
are the same sweep — one row per thread, the reference subtraction order,
dependencies awaited through mailbox packets — so they stay bitwise
identical to each other and to the reference.  Each function keeps the
reference's argument validation and error behaviour.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import device as dv
from .csr import lower_pattern
from .errors import ConfigurationError, ZeroPivotError
from .lower import TileLayout, er_chunks
from .ordering import LevelSchedule, StagePartition, compute_levels, compute_levels_backward
from .symbolic import IluFactors
from .sync import SyncSchedule, build_sync_schedule, build_triangle_schedule

__all__ = [
    "FORWARD",
    "BACKWARD",
    "solve_serial",
    "solve_baseline_csrls",
    "solve_ls",
    "solve_ls_lower",
    "apply_preconditioner",
    "SolveSetup",
    "build_solve_setup",
]

FORWARD = "forward"
BACKWARD = "backward"


def _check_which(which: str) -> None:
    if which not in (FORWARD, BACKWARD):
        raise ValueError(f"which must be 'forward' or 'backward', got {which!r}")


def _check_schedule(factors: IluFactors, schedule, partition=None) -> None:
    """The GPU sweeps do not read the CPU wait lists, but a schedule (or
    partition) built for another matrix is still an error, as it would be
    for the reference's kernels that index by it."""
    if schedule is not None and np.asarray(schedule.owner).size != factors.n:
        raise ConfigurationError("sync schedule does not match the factors")
    if partition is not None and partition.n != factors.n:
        raise ConfigurationError("stage partition does not match the factors")


def _device_sweep(factors: IluFactors, b: np.ndarray, which: str) -> np.ndarray:
    if factors.n == 0:
        return np.array(b, dtype=np.float64, copy=True)
    d = factors.upload_values()
    if which == BACKWARD:
        bad = d.first_zero_diag()
        if bad >= 0:
            raise ZeroPivotError(bad)
    x = dv.upload_vec(b, factors.n)
    d.solve_async(0 if which == FORWARD else 1, x, x)
    dv.check_hang()
    return dv.download_vec(x, factors.n)


def solve_serial(factors: IluFactors, b: np.ndarray, which: str) -> np.ndarray:
    """Forward (unit L) or backward (U) sweep (trisolve.py:60-71)."""
    _check_which(which)
    return _device_sweep(factors, b, which)


def solve_baseline_csrls(
    factors: IluFactors,
    b: np.ndarray,
    schedule: LevelSchedule,
    nthreads: int,
    which: str,
) -> np.ndarray:
    """The paper's CSR-LS baseline (trisolve.py:74-108): one level at a time,
    here one kernel launch per level replayed from a CUDA graph
    (jv_solve_level) — the GPU counterpart of the reference's barrier per
    level, kept for comparison with the sync-free and region sweeps."""
    _check_which(which)
    if schedule.n != factors.n:
        raise ConfigurationError("level schedule does not match the factors")
    if factors.n == 0:
        return np.array(b, dtype=np.float64, copy=True)
    d = factors.upload_values()
    if which == BACKWARD:
        bad = d.first_zero_diag()
        if bad >= 0:
            raise ZeroPivotError(bad)
    x = dv.upload_vec(b, factors.n)
    d.solve_csrls_async(0 if which == FORWARD else 1, x, x)
    return dv.download_vec(x, factors.n)


def solve_ls(
    factors: IluFactors,
    b: np.ndarray,
    schedule: SyncSchedule,
    which: str,
) -> np.ndarray:
    """Point-to-point solve entry point (trisolve.py:111-137)."""
    _check_which(which)
    _check_schedule(factors, schedule)
    return _device_sweep(factors, b, which)


def solve_ls_lower(
    factors: IluFactors,
    b: np.ndarray,
    schedule: SyncSchedule,
    partition: StagePartition,
    lower_layout,
    which: str,
    nthreads: int | None = None,
) -> np.ndarray:
    """Two-stage solve entry point (trisolve.py:140-182)."""
    _check_which(which)
    _check_schedule(factors, schedule, partition)
    return _device_sweep(factors, b, which)


@dataclass
class SolveSetup:
    """Prebuilt schedules for one solve path (trisolve.py:185-198)."""

    path: str
    nthreads: int = 1
    fwd_levels: LevelSchedule | None = None
    bwd_levels: LevelSchedule | None = None
    fwd_sync: SyncSchedule | None = None
    bwd_sync: SyncSchedule | None = None
    upper_sync: SyncSchedule | None = None
    partition: StagePartition | None = None
    lower_layout: object = None
    extra: dict = field(default_factory=dict)


def build_solve_setup(
    factors: IluFactors,
    path: str,
    nthreads: int = 1,
    partition: StagePartition | None = None,
    lower_layout=None,
) -> SolveSetup:
    """Schedules per path (trisolve.py:201-228); levels on the GPU."""
    pat = factors.pattern
    setup = SolveSetup(path, nthreads, partition=partition, lower_layout=lower_layout)
    if path == "serial":
        return setup
    if path == "csrls":
        setup.fwd_levels = compute_levels(lower_pattern(pat))
        setup.bwd_levels = compute_levels_backward(pat)
        return setup
    if path == "ls":
        setup.fwd_sync = build_triangle_schedule(pat, nthreads, FORWARD)
        setup.bwd_sync = build_triangle_schedule(pat, nthreads, BACKWARD)
        return setup
    if path == "ls_lower":
        if partition is None:
            raise ConfigurationError("ls_lower needs the stage partition")
        setup.upper_sync = build_sync_schedule(partition, pat, nthreads)
        setup.bwd_sync = build_triangle_schedule(pat, nthreads, BACKWARD)
        if lower_layout is None:
            setup.lower_layout = er_chunks(pat, partition.n_upper, nthreads)
        return setup
    raise ConfigurationError(f"unknown solve path {path!r}")


def apply_preconditioner(
    factors: IluFactors, r: np.ndarray, setup: SolveSetup | None = None
) -> np.ndarray:
    """z = U^-1 (L^-1 r) (trisolve.py:231-249): both sweeps back to back on
    the device, one upload and one download."""
    if setup is not None and setup.path not in ("serial", "csrls", "ls", "ls_lower"):
        raise ConfigurationError(f"unknown solve path {setup.path!r}")
    if factors.n == 0:
        return np.array(r, dtype=np.float64, copy=True)
    d = factors.upload_values()
    x = dv.upload_vec(r, factors.n)
    d.solve_async(0, x, x)
    bad = d.first_zero_diag()
    if bad >= 0:
        raise ZeroPivotError(bad)
    d.solve_async(1, x, x)
    dv.check_hang()
    return dv.download_vec(x, factors.n)
