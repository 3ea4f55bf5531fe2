"""Numeric ILU(k, tau) factorization — the reference factor.py API
(/root/reference/pkg/src/ilukit/factor.py) backed by the sync-free sm_100a
kernel jv_factor.

Every path computes the reference's per-row up-looking elimination in
ascending pivot order with separately rounded binary64 ops, so results are
bitwise equal to the reference factor_serial (_kernels.py:197-204).  A zero
post-elimination diagonal is reported as the smallest such row, after the
kernel has quiesced (factor.py:61-63).
"""

from __future__ import annotations

import numpy as np

from . import device as dv
from .errors import ZeroPivotError
from .symbolic import IluFactors

__all__ = ["factor_serial", "factor_parallel_upper", "row_inf_norms"]


def row_inf_norms(factors: IluFactors) -> np.ndarray:
    """Inf-norm of each row's current values (zeros unless tau > 0); the
    tau drop threshold is relative to these (factor.py:25-34)."""
    if factors.n == 0:
        return np.zeros(0)
    d = factors.upload_values()
    d.compute_norms()
    return dv.host_f64(d.norms, factors.n)


def _run(factors: IluFactors, lo=0, hi=None, ready_below=0, keep_after_bad=False) -> int:
    d = factors.upload_values()
    bad = d.factor(lo, hi, ready_below)
    n_out = factors.pattern.nnz
    if bad >= 0 and keep_after_bad:
        # the reference stops at the first zero pivot: rows after it keep
        # their input values, which the host array still holds
        n_out = int(factors.pattern.row_start[bad + 1])
    factors.val = np.ascontiguousarray(factors.val, dtype=np.float64)
    dv.download_f64(factors.val, d.val, n_out)
    return bad


def factor_serial(factors: IluFactors) -> None:
    """Up-looking ILU over all rows, in place; ZeroPivotError(first row).

    The device sweeps every row; as the reference stops at the first zero
    pivot, only the rows up to it are copied back, so the observable state
    matches the reference's."""
    if factors.n == 0:
        return
    factors.val = np.ascontiguousarray(factors.val, dtype=np.float64)
    if factors.pattern.nnz * 8 >= dv.STREAM_MIN_BYTES and dv.pinned_host(factors.val):
        # large page-locked host values: upload, factorization and download
        # overlap chunk by chunk (DevIlu.factor_streamed)
        d = factors.device()
        bad = d.factor_streamed(factors.val)
        d.holder = factors
    else:
        bad = _run(factors, keep_after_bad=True)
    if bad >= 0:
        raise ZeroPivotError(int(bad))


def _row_range(rows: np.ndarray, n: int):
    """[lo, hi) when `rows` is exactly a contiguous index range."""
    if rows.size == 0:
        return 0, 0
    lo, hi = int(rows.min()), int(rows.max()) + 1
    if hi - lo == rows.size and np.unique(rows).size == rows.size:
        return lo, hi
    return None


def factor_parallel_upper(factors: IluFactors, schedule) -> None:
    """Factor the scheduled (upper-stage) rows (factor.py:48-63).

    The point-to-point waits of `schedule` are not needed on the GPU: each
    row awaits its own pivots through the mailbox, in any order; only the
    row set matters."""
    rows = np.asarray(schedule.order, dtype=np.int64)
    if factors.n == 0 or rows.size == 0:
        return
    rng = _row_range(rows, factors.n)
    if rng is None:
        raise NotImplementedError("factor_parallel_upper: schedule rows must form an index range")
    lo, hi = rng
    bad = _run(factors, lo, hi, ready_below=lo)
    if bad >= 0:
        raise ZeroPivotError(int(bad))
