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

import os
import time

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


def _host_values(factors: IluFactors) -> np.ndarray:
    """The caller's value array as contiguous float64 (replaced in the
    factors only when it is not already), without counting as a read."""
    host = factors._host()
    if not (isinstance(host, np.ndarray) and host.dtype == np.float64
            and host.flags.c_contiguous):
        factors.val = np.ascontiguousarray(host, dtype=np.float64)
        host = factors._host()
    return host


def _run(factors: IluFactors, lo=0, hi=None, ready_below=0, keep_after_bad=False) -> int:
    d = factors.upload_values()
    bad = d.factor(lo, hi, ready_below)
    n_out = factors.pattern.nnz
    if bad >= 0 and keep_after_bad:
        # the reference stops at the first zero pivot: rows after it keep
        # their input values, which the host array still holds
        n_out = int(factors.pattern.row_start[bad + 1])
    host = _host_values(factors)
    dv.download_f64(host, d.val, n_out)
    if n_out == factors.pattern.nnz:
        factors._synced()   # host and device hold the same factors now
    else:
        factors._dirty = True
    return bad


def factor_serial(factors: IluFactors) -> None:
    """Up-looking ILU over all rows, in place; ZeroPivotError(first row).

    The device sweeps every row; as the reference stops at the first zero
    pivot, only the rows up to it are copied back, so the observable state
    matches the reference's."""
    if factors.n == 0:
        return
    host = _host_values(factors)
    if (factors.pattern.nnz * 8 >= dv.STREAM_MIN_BYTES and not factors.device_is_current()
            and dv.pinned_host(host)):
        # large page-locked host values: upload, factorization and download
        # can overlap chunk by chunk (DevIlu.factor_streamed).  The chunked
        # sweeps run the sync-free kernel per row range, which for some
        # patterns costs more than the overlap saves (config 3: 19 vs 8 ms),
        # so both ways are timed once per pattern and the faster one kept
        # (identical results).
        d = factors.device()
        mode = _stream_mode(d)
        t0 = time.perf_counter()
        if mode == "streamed":
            bad = d.factor_streamed(host)
            d.holder = factors
            if bad < 0:
                factors._synced()
            else:
                factors._dirty = True
        else:
            bad = _run(factors, keep_after_bad=True)
        _stream_note(d, mode, time.perf_counter() - t0)
    else:
        bad = _run(factors, keep_after_bad=True)
    if bad >= 0:
        raise ZeroPivotError(int(bad))


# calls 1-2 whole (the first builds schedules), 3-4 streamed (the third builds
# the chunk schedules); from the fifth call on the faster of calls 2 and 4
_STREAM_PLAN = ("whole", "whole", "streamed", "streamed")


def _stream_mode(d) -> str:
    forced = os.environ.get("JV_STREAM")           # "0" whole, "1" streamed
    if forced in ("0", "1"):
        return "streamed" if forced == "1" else "whole"
    hist = d.__dict__.setdefault("_stream_hist", [])
    if len(hist) < len(_STREAM_PLAN):
        return _STREAM_PLAN[len(hist)]
    return "streamed" if hist[3] < hist[1] else "whole"


def _stream_note(d, mode: str, seconds: float) -> None:
    hist = d.__dict__.setdefault("_stream_hist", [])
    if len(hist) < len(_STREAM_PLAN):
        hist.append(seconds)


def _row_runs(rows: np.ndarray):
    """The maximal runs [lo, hi) of consecutive indices in the row set."""
    r = np.unique(rows)
    if r.size == 0:
        return []
    brk = np.flatnonzero(np.diff(r) != 1)
    los = np.concatenate(([r[0]], r[brk + 1]))
    his = np.concatenate((r[brk] + 1, [r[-1] + 1]))
    return [(int(a), int(b)) for a, b in zip(los, his)]


def factor_parallel_upper(factors: IluFactors, schedule) -> None:
    """Factor the scheduled (upper-stage) rows (factor.py:48-63).

    The point-to-point waits of `schedule` are not needed on the GPU: each
    row awaits its own pivots through the mailbox, in any order; only the
    row set matters.  Rows outside the set are read as they are (the
    reference's kernels never wait for them either): the set is factored
    run by run of consecutive rows in ascending order, each launch taking
    everything below its run as final — one launch for the usual upper
    block [0, n_upper)."""
    rows = np.asarray(schedule.order, dtype=np.int64)
    if factors.n == 0 or rows.size == 0:
        return
    runs = _row_runs(rows)
    if len(runs) == 1:
        lo, hi = runs[0]
        bad = _run(factors, lo, hi, ready_below=lo)
    else:
        d = factors.upload_values()
        bad = -1
        for lo, hi in runs:
            b = d.factor(lo, hi, lo)
            if b >= 0 and bad < 0:
                bad = b
        dv.download_f64(_host_values(factors), d.val, factors.pattern.nnz)
        factors._synced()
    if bad >= 0:
        raise ZeroPivotError(int(bad))
