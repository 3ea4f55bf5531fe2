"""Generate the golden fixtures by running the REFERENCE itself.

Run in the build container, where the reference package is importable from
/root/reference/pkg/src (numba present).  Outputs (committed):

  tests/golden/small.npz         full input/output arrays for small cases
  tests/golden/full_digests.json sha256 digests + stats of the five
                                 BASELINE configs at published size

Nothing at test or bench time reads /root/reference; only these files.

    python tests/golden/make_golden.py [--small] [--full c1,c2,...]
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

import ilukit as ik  # noqa: E402  (the reference)
from ilukit.ordering import LOWER_A_PLUS_AT  # noqa: E402
from ilukit.trisolve import BACKWARD, FORWARD  # noqa: E402


def digest(a, kind):
    a = np.ascontiguousarray(np.asarray(a), dtype=np.int64 if kind == "i" else np.float64)
    return hashlib.sha256(a.tobytes()).hexdigest()


def to_ref(m):
    return ik.CsrMatrix(m.n, m.row_start.copy(), m.col.copy(), m.val.copy())


# ---------------------------------------------------------------- small


def small_cases():
    """(name, reference matrix, k, tau, milu, cut) — cut=None: default rule"""
    cases = [
        ("kat2", ik.CsrMatrix.from_dense([[4.0, 2.0], [1.0, 3.0]]), 0, 0.0, False, None),
        ("kat3_fill_dropped", ik.CsrMatrix.from_dense([[2.0, 0.0, 1.0], [1.0, 2.0, 0.0],
                                                        [0.0, 1.0, 2.0]]), 0, 0.0, False, None),
        ("zero_pivot_row1", ik.CsrMatrix.from_dense([[2.0, 4.0], [1.0, 2.0]]), 0, 0.0, False, None),
        ("fma_probe", ik.CsrMatrix.from_dense([[1.0, 1.0 + 2.0 ** -30],
                                               [1.0 + 2.0 ** -30, 1.0 + 2.0 ** -29]]),
         0, 0.0, False, None),
        ("tridiag32", ik.tridiag(32), 0, 0.0, False, None),
        ("poisson2d_8", ik.poisson2d(8), 0, 0.0, False, None),
        ("poisson2d_16_cut2", ik.poisson2d(16), 0, 0.0, False, 2),
        ("poisson2d_4_ilu1", ik.poisson2d(4), 1, 0.0, False, None),
        ("poisson2d_4_ilu2", ik.poisson2d(4), 2, 0.0, False, None),
        ("poisson2d_4_milu", ik.poisson2d(4), 0, 0.0, True, None),
        ("poisson3d_5", ik.poisson3d(5), 0, 0.0, False, None),
        ("poisson3d_6_ilu1", ik.poisson3d(6), 1, 0.0, False, None),
        ("convdiff2d_12_ilu1", ik.convdiff2d(12, seed=3), 1, 0.0, False, None),
        ("convdiff2d_12_ilu1_tau", ik.convdiff2d(12, seed=3), 1, 1e-2, False, None),
        ("rdd40_tau", ik.random_diag_dominant(40, row_nnz=6, seed=7), 0, 0.05, False, None),
        ("rdd40_tau_milu", ik.random_diag_dominant(40, row_nnz=6, seed=7), 0, 0.05, True, None),
        ("rdd150_tau_milu_cut3", ik.random_diag_dominant(150, row_nnz=6, seed=12), 0, 0.05,
         True, 3),
        ("rdd200_cut4", ik.random_diag_dominant(200, row_nnz=7, seed=9), 0, 0.0, False, 4),
        ("rdd300_sym", ik.random_diag_dominant(300, row_nnz=6, seed=41, symmetric_pattern=True),
         0, 0.0, False, None),
        ("rdd300_ilu2", ik.random_diag_dominant(300, row_nnz=5, seed=5), 2, 0.0, False, None),
    ]
    for seed in range(12):
        n = 60 + (seed * 97) % 241
        cases.append((f"suite{seed}", ik.random_diag_dominant(
            n, row_nnz=4 + seed % 5, seed=seed, symmetric_pattern=bool(seed % 2)),
            seed % 3 == 0 and 1 or 0, 0.0, False, None))
    return cases


def run_reference(a, k, tau, milu, cut, base=None, min_level_rows=16, density=4.0, rhs_seed=0):
    """The reference front end + factor + solves + spmv; returns arrays."""
    n = a.n
    base = base if base is not None else ik.Permutation.identity(n)
    pa = ik.permute_symmetric(a, base)
    src = ik.lower_pattern(ik.symmetrize_pattern(pa.pattern))
    sched = ik.compute_levels(src, LOWER_A_PLUS_AT)
    cfg = ik.PartitionConfig(min_level_rows, density)
    if cut is None:
        part = ik.partition_stages(sched, np.diff(pa.row_start), cfg)
    else:
        levels = sched.levels
        upper = [r.copy() for r in levels[:cut]]
        lower = (np.concatenate([levels[i] for i in range(cut, len(levels))])
                 if cut < len(levels) else np.zeros(0, dtype=np.int64))
        part = ik.StagePartition(upper, lower, cut, cfg, LOWER_A_PLUS_AT)
    lperm = ik.build_level_permutation(part)
    total = lperm.compose(base)
    permuted = ik.permute_symmetric(a, total)
    pattern, fill = ik.iluk_pattern(permuted.pattern, k)
    factors = ik.assemble_factors(a, pattern, total, tau, milu)
    assembled = factors.val.copy()
    from ilukit.factor import row_inf_norms
    norms = row_inf_norms(factors)
    bad = -1
    try:
        ik.factor_serial(factors)
    except ik.ZeroPivotError as e:
        bad = e.row
    rng = np.random.default_rng(rhs_seed)
    b0 = rng.uniform(-1.0, 1.0, n)
    b = b0[total.perm]
    y = ik.solve_serial(factors, b, FORWARD)
    try:
        x = ik.solve_serial(factors, y, BACKWARD)
        xbad = -1
    except ik.ZeroPivotError as e:
        x, xbad = np.zeros(n), e.row
    spmv_y = ik.spmv(permuted, b)
    spmv_a = ik.spmv(a, b0)
    fwd_lev = ik.compute_levels(ik.lower_pattern(pattern)).level_of
    bwd_lev = ik.compute_levels_backward(pattern).level_of
    sym = ik.symmetrize_pattern(a.pattern)
    low = ik.lower_pattern(sym)
    return dict(
        a_rs=a.row_start, a_col=a.col, a_val=a.val, base=base.perm,
        sym_rs=sym.row_start, sym_col=sym.col, low_rs=low.row_start, low_col=low.col,
        level_of=sched.level_of, cut=np.int64(part.cut_level), n_upper=np.int64(part.n_upper),
        perm=total.perm, p_rs=permuted.row_start, p_col=permuted.col, p_val=permuted.val,
        f_rs=pattern.row_start, f_col=pattern.col, fill=fill.level, diag=factors.diag_pos,
        assembled=assembled, norms=norms, fval=factors.val, bad=np.int64(bad),
        b0=b0, b=b, y=y, x=x, xbad=np.int64(xbad), spmv_perm=spmv_y, spmv_a=spmv_a,
        fwd_lev=fwd_lev, bwd_lev=bwd_lev,
        k=np.int64(k), tau=np.float64(tau), milu=np.int64(milu),
    )


def make_small(path):
    out = {}
    names = []
    for name, a, k, tau, milu, cut in small_cases():
        res = run_reference(a, k, tau, milu, cut)
        if a.n <= 400:
            res["rcm"] = ik.rcm_order(a.pattern).perm
        for key, v in res.items():
            out[f"{name}/{key}"] = np.asarray(v)
        names.append(name)
    out["_names"] = np.array(names)
    np.savez_compressed(path, **out)
    print(f"wrote {path}: {len(names)} cases, {os.path.getsize(path)} bytes")


# ----------------------------------------------------------------- full


def make_full(path, which, c5_seeds=(0, 1)):
    from paper_1812_06160_b200 import workloads as W

    result = json.load(open(path)) if os.path.exists(path) else {}
    for cfg in which:
        t0 = time.time()
        s = W.CONFIGS[cfg]
        mats = []
        if cfg == "c5":
            for seed in c5_seeds:
                mats.append((f"c5_seed{seed}", W.rmat(18, seed), None))
        else:
            a, base, _ = W.config_matrix(cfg)
            ref = to_ref(a)
            if base == "rcm":
                tb = time.time()
                bperm = ik.rcm_order(ref.pattern)
                print(f"  {cfg} rcm {time.time() - tb:.1f}s")
            elif base is None:
                bperm = None
            else:
                bperm = ik.Permutation(base.perm)
            mats.append((cfg, a, bperm))
        for key, a, bperm in mats:
            ref = to_ref(a)
            res = run_reference(ref, s["k"], s["tau"], False, None, base=bperm,
                                min_level_rows=s["min_level_rows"])
            ints = ["base", "sym_rs", "sym_col", "low_rs", "low_col", "level_of", "perm", "p_rs",
                    "p_col", "f_rs", "f_col", "fill", "diag", "fwd_lev", "bwd_lev"]
            flts = ["p_val", "assembled", "norms", "fval", "b", "y", "x", "spmv_perm", "spmv_a"]
            d = {k: digest(res[k], "i") for k in ints}
            d.update({k: digest(res[k], "f") for k in flts})
            low = res["f_col"] < np.repeat(np.arange(a.n), np.diff(res["f_rs"]))
            stats = dict(
                n=int(a.n), nnz=int(a.nnz), nnz_f=int(res["f_col"].size),
                nnz_l=int(low.sum()), nlev=int(res["level_of"].max() + 1),
                cut=int(res["cut"]), n_upper=int(res["n_upper"]), bad=int(res["bad"]),
                xbad=int(res["xbad"]), fwd_depth=int(res["fwd_lev"].max() + 1),
                bwd_depth=int(res["bwd_lev"].max() + 1),
                dropped=int(np.sum((res["fval"] == 0.0) & low & (res["assembled"] != 0.0))),
                # L positions left exactly 0 (dropped multipliers, fill included)
                zero_l=int(np.sum((res["fval"] == 0.0) & low)),
                k=s["k"], tau=s["tau"], min_level_rows=s["min_level_rows"],
                x_absmax=float(np.max(np.abs(res["x"]))),
                fval_absmax=float(np.max(np.abs(res["fval"]))),
            )
            result[key] = dict(digests=d, stats=stats)
            print(f"{key}: {stats} ({time.time() - t0:.1f}s)")
            json.dump(result, open(path, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--small", action="store_true")
    ap.add_argument("--full", default="")
    ap.add_argument("--c5-seeds", default="0-1", help="R-MAT seeds for c5, e.g. 0-63")
    ap.add_argument("--out", default=os.path.join(HERE, "full_digests.json"))
    args = ap.parse_args()
    lo, _, hi = args.c5_seeds.partition("-")
    seeds = range(int(lo), int(hi or lo) + 1)
    if args.small:
        make_small(os.path.join(HERE, "small.npz"))
    if args.full:
        make_full(args.out, args.full.split(","), seeds)
