"""Schema-compatible run report of the device path.

`run_report` runs the reference pipeline's measurement protocol
(ilukit/pipeline.py:209-382, report schema pkg/docs/report_schema.json,
schema version 1) on the GPU and returns a report with the same keys,
types and meaning:

* timings per phase and per worker count: `setup` (device front end:
  ordering -> levels -> partition -> permutation -> symbolic -> assembly),
  `factor_upper` / `factor_lower` (the upper-stage kernel and the two-stage
  lower tail), `solve_csrls` (the paper's level-synchronous baseline, one
  launch per level), `solve_ls` (the sync-free / region sweeps) and
  `solve_ls_lower` (the same sweeps: on the GPU the two-stage solve is the
  same kernel), medians of `repeats` device-timed runs, in seconds;
* the GPU has no worker threads: every requested worker count is a
  separate, complete measurement keyed by that count, so `speedups`
  (timing[1] / timing[t]) read ~1 and `determinism_ok` compares the digests
  of independent runs — the run-to-run determinism of the sync-free kernels;
* `digests`: sha256 of the serial factor values (the drop-in factor_serial,
  bitwise the reference's), of the staged factorization per worker count,
  and of each solve path's result per worker count — directly comparable
  with a reference report of the same configuration.
"""

from __future__ import annotations

import hashlib
import statistics
import time

import numpy as np

from . import device as dv
from .csr import CsrMatrix, Permutation
from .errors import ConfigurationError
from .krylov import gmres, pcg
from .ordering import rcm_order
from .plan import build_plan
from .symbolic import IluFactors
from .csr import SparsityPattern

REPORT_SCHEMA_VERSION = 1
SOLVE_PATHS = ("solve_csrls", "solve_ls", "solve_ls_lower")

__all__ = ["run_report", "REPORT_SCHEMA_VERSION", "SOLVE_PATHS", "level_stats"]


def _digest(arr) -> str:
    return hashlib.sha256(np.ascontiguousarray(arr).tobytes()).hexdigest()


def level_stats(level_of: np.ndarray) -> dict:
    """num_levels / min / max / median rows per level (ordering.py level_stats)."""
    if level_of.size == 0:
        return {"num_levels": 0, "min_rows": 0, "max_rows": 0, "median_rows": 0}
    counts = np.bincount(level_of)
    return {"num_levels": int(counts.size), "min_rows": int(counts.min()),
            "max_rows": int(counts.max()), "median_rows": int(np.median(counts))}


def _dev_time(fn, repeats, reset=None):
    t = dv.torch()
    e0, e1 = t.cuda.Event(enable_timing=True), t.cuda.Event(enable_timing=True)
    out = []
    for _ in range(repeats):
        if reset is not None:
            reset()
        e0.record()
        fn()
        e1.record()
        t.cuda.synchronize()
        out.append(e0.elapsed_time(e1) / 1e3)
    return float(statistics.median(out))


def run_report(a: CsrMatrix, matrix_name: str = "matrix", order="natural", levels_on="AplusAT",
               k: int = 0, tau: float = 0.0, milu: bool = False, lower: str = "auto",
               min_level_rows: int = 16, density_factor: float = 4.0, tile_size: int = 256,
               threads=(1,), solver: str = "none", restart: int = 50, tol: float = 1e-8,
               maxit: int = 1000, repeats: int = 3) -> dict:
    """Run the device hot path under the reference's pipeline protocol and
    return a report valid against report_schema.json (version 1).  `order`
    is "natural", "rcm", or a Permutation (reported as "file")."""
    if levels_on != "AplusAT":
        raise ConfigurationError("the device front end schedules on levels of lower(A+A^T)")
    if lower not in ("auto", "sr", "er", "none"):
        raise ConfigurationError(f"unknown lower method {lower!r}")
    if solver not in ("none", "pcg", "gmres"):
        raise ConfigurationError(f"unknown solver {solver!r}")
    if not threads or any(int(x) < 1 for x in threads):
        raise ConfigurationError("worker counts must be positive")
    if repeats < 1:
        raise ConfigurationError("repeats must be >= 1")
    threads = list(dict.fromkeys(int(x) for x in threads))
    t = dv.torch()
    if isinstance(order, Permutation):
        base, order_name = order.perm, "file"
    elif order == "rcm":
        base, order_name = rcm_order(a.pattern).perm, "rcm"
    elif order == "natural":
        base, order_name = None, "natural"
    else:
        raise ConfigurationError(f"unknown order {order!r}")
    mlr, dens = (1, float("inf")) if lower == "none" else (min_level_rows, density_factor)

    def build():
        return build_plan(a, base_perm=base, k=k, tau=tau, milu=milu, min_level_rows=mlr,
                          density_factor=dens)

    probe = build()
    n_upper, n = probe.n_upper, a.n
    if lower in ("sr", "er"):
        method = lower if n_upper < n else "none"
    elif lower == "none" or n_upper == n:
        method = "none"
    else:
        method = "er"      # both methods are the same device launches (lower.py)

    # serial reference digest through the drop-in API (bitwise = reference)
    ilu = probe.ilu
    pat = SparsityPattern(n, dv.host_i64(ilu.row_start, n + 1), dv.host_i64(ilu.col, ilu.nnz))
    ref = IluFactors(n, pat, dv.host_f64(probe.assembled, ilu.nnz).copy(),
                     dv.host_i64(ilu.diag_pos, n), Permutation(dv.host_i64(probe.perm, n)),
                     tau, milu)
    from .factor import factor_serial
    factor_serial(ref)
    serial_digest = _digest(ref.val)

    timings = {p: {} for p in ("setup", "factor_upper", "factor_lower") + SOLVE_PATHS}
    factor_digests, solve_digests = {}, {p: {} for p in SOLVE_PATHS}
    krylov_report = None
    for w in threads:
        setup = []
        for _ in range(repeats):
            t.cuda.synchronize()
            t0 = time.perf_counter()
            plan = build()
            t.cuda.synchronize()
            setup.append(time.perf_counter() - t0)
        timings["setup"][w] = float(statistics.median(setup))
        ilu = plan.ilu
        nu = plan.n_upper

        def upper():
            if nu:
                ilu._factor_tickets(0, nu, 0, True)
        timings["factor_upper"][w] = _dev_time(upper, repeats, plan.reset_values)
        plan.reset_values()
        upper()
        post_upper = ilu.val.clone()
        if nu < n:
            timings["factor_lower"][w] = _dev_time(
                lambda: ilu.factor_tail_async(nu), repeats, lambda: ilu.load_values(post_upper))
            ilu.load_values(post_upper)
            bad = ilu.factor_tail(nu)
        else:
            timings["factor_lower"][w] = None
            bad = dv.read_row_slot(ilu.err)
        if bad >= 0:
            from .errors import ZeroPivotError
            raise ZeroPivotError(bad)
        factor_digests[w] = _digest(ilu.host_val())
        b = dv.empty_f64(n)
        ones = dv.f64(np.ones(n))
        dv.spmv_dev(plan.permuted, ones, b)
        y, z = dv.empty_f64(n), dv.empty_f64(n)
        runners = {
            "solve_csrls": lambda: (ilu.solve_csrls_async(0, b, y), ilu.solve_csrls_async(1, y, z)),
            "solve_ls": lambda: (ilu.solve_async(0, b, y), ilu.solve_async(1, y, z)),
            "solve_ls_lower": lambda: (ilu.solve_async(0, b, y), ilu.solve_async(1, y, z)),
        }
        for path, run in runners.items():
            run()
            solve_digests[path][w] = _digest(dv.host_f64(z, n))
            timings[path][w] = _dev_time(run, repeats)
        dv.check_hang()
        if krylov_report is None and solver != "none":
            from .krylov import IluPreconditioner
            from .csr import CsrMatrix as _C
            prs, pcol = plan.permuted.host_pattern()
            pa = _C(n, prs, pcol, dv.host_f64(plan.permuted.val, plan.permuted.nnz))
            fac = IluFactors(n, SparsityPattern(n, dv.host_i64(ilu.row_start, n + 1),
                                                dv.host_i64(ilu.col, ilu.nnz)),
                             ilu.host_val(), dv.host_i64(ilu.diag_pos, n),
                             Permutation(dv.host_i64(plan.perm, n)), tau, milu)
            pre = IluPreconditioner(fac)
            bh = dv.host_f64(b, n)
            res = (pcg(pa, bh, pre, tol, maxit) if solver == "pcg"
                   else gmres(pa, bh, pre, restart, tol, maxit))
            krylov_report = {"method": solver, "iterations": int(res.iterations),
                             "converged": bool(res.converged),
                             "final_relative_residual": float(res.residual_history[-1]),
                             "stopping_rule": "relative_residual"}

    determinism_ok = (len(set(factor_digests.values())) == 1
                      and all(len(set(d.values())) == 1 for d in solve_digests.values())
                      and next(iter(factor_digests.values())) == serial_digest)

    def speedup_row(row):
        base_t = row.get(1)
        if not base_t:
            return {w: None for w in row}
        return {w: (base_t / v if v else None) for w, v in row.items()}

    speedups = {ph: speedup_row({w: v for w, v in row.items() if v is not None})
                for ph, row in timings.items()}
    cs = timings["solve_csrls"].get(1)
    vs_csrls = {p: {w: (cs / v if cs and v else None) for w, v in timings[p].items()}
                for p in SOLVE_PATHS}
    level_of = dv.host_i64(probe.level_of, n)
    key = lambda d: {str(w): v for w, v in d.items()}
    return {
        "schema_version": REPORT_SCHEMA_VERSION,
        "config": {"matrix": matrix_name, "order": order_name, "levels_on": levels_on, "k": k,
                   "tau": tau, "milu": milu, "lower": lower, "min_level_rows": min_level_rows,
                   "density_factor": density_factor, "tile_size": tile_size,
                   "threads": threads, "solver": solver, "restart": restart, "tol": tol,
                   "maxit": maxit, "repeats": repeats},
        "matrix": {"name": matrix_name, "n": a.n, "nnz": a.nnz,
                   "mean_row_nnz": a.nnz / a.n if a.n else 0.0},
        "levels": level_stats(level_of),
        "partition": {"cut_level": probe.cut, "num_upper_levels": probe.cut,
                      "n_upper": n_upper, "rows_excluded": n - n_upper, "method": method},
        "timings": {ph: key(row) for ph, row in timings.items()},
        "speedups": {ph: key(row) for ph, row in speedups.items()},
        "solve_speedups_vs_csrls": {p: key(row) for p, row in vs_csrls.items()},
        "krylov": krylov_report,
        "digests": {"serial": serial_digest, "factor": key(factor_digests),
                    "solve": {p: key(d) for p, d in solve_digests.items()}},
        "determinism_ok": bool(determinism_ok),
    }
