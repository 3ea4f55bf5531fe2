"""Drop-in calls keep the factor values resident in HBM between calls (the
reference's Krylov pattern `precond = lambda r: apply_preconditioner(factors,
r)`, pipeline.py:300 / krylov.py:200) — and never serve stale values: any
way the caller can have changed the host array forces a fresh upload.  Also
factor_parallel_upper over a schedule whose rows are not one index range
(factor.py:48-63: rows outside the schedule are read as they are)."""

import types

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

jv = pytest.importorskip("paper_1812_06160_b200")
from paper_1812_06160_b200 import device as dv  # noqa: E402


def make(n=24):
    a = jv.poisson2d(n)
    f = jv.assemble_factors(a, jv.ilu0_pattern(a.pattern), jv.Permutation.identity(a.n))
    return a, f


@pytest.fixture
def uploads(monkeypatch):
    """Counts whole-array value uploads."""
    calls = []
    real = dv.upload_f64

    def counted(dst, src):
        calls.append(int(np.asarray(src).size))
        return real(dst, src)

    monkeypatch.setattr(dv, "upload_f64", counted)
    return calls


def expected_apply(f, vals, r):
    rs = f.pattern.row_start.astype(np.int64)
    col = f.pattern.col.astype(np.int64)
    diag = f.diag_pos.astype(np.int64)
    y = oracle.solve_forward(rs, col, vals, r)
    x, _ = oracle.solve_backward(rs, col, vals, diag, y)
    return x


def test_preconditioner_lambda_uploads_once(uploads, rng):
    a, f = make()
    jv.factor_serial(f)
    uploads.clear()
    precond = lambda r: jv.apply_preconditioner(f, r)  # noqa: E731
    want_vals = f.val.copy()          # a read: the next call must upload
    outs = [precond(rng.uniform(-1, 1, a.n)) for _ in range(5)]
    assert len(uploads) == 1, uploads
    r = rng.uniform(-1, 1, a.n)
    assert np.array_equal(precond(r), expected_apply(f, want_vals, r))
    assert len(uploads) == 1
    assert all(np.isfinite(o).all() for o in outs)


def test_factor_then_solve_needs_no_upload(uploads, rng):
    a, f = make()
    jv.factor_serial(f)
    n_up = len(uploads)
    b = rng.uniform(-1, 1, a.n)
    y = jv.solve_serial(f, b, "forward")
    x = jv.solve_serial(f, y, "backward")
    assert len(uploads) == n_up          # the factors never left the device
    assert np.array_equal(x, expected_apply(f, f.val, b))


def test_write_through_attribute_is_seen(rng):
    a, f = make()
    jv.factor_serial(f)
    r = rng.uniform(-1, 1, a.n)
    jv.apply_preconditioner(f, r)
    f.val[f.diag_pos] *= 2.0          # in-place edit through the attribute
    vals = f.val.copy()
    assert np.array_equal(jv.apply_preconditioner(f, r), expected_apply(f, vals, r))


def test_kept_alias_is_seen(rng):
    a, f = make()
    alias = f.val                     # a reference the caller keeps
    view = alias[3:]
    jv.factor_serial(f)
    r = rng.uniform(-1, 1, a.n)
    jv.apply_preconditioner(f, r)
    view[0] = view[0] * 3.0           # no attribute access at all
    vals = alias.copy()
    assert np.array_equal(jv.apply_preconditioner(f, r), expected_apply(f, vals, r))


def test_replaced_array_is_seen(rng):
    a, f = make()
    jv.factor_serial(f)
    r = rng.uniform(-1, 1, a.n)
    jv.apply_preconditioner(f, r)
    vals = f.val * 0.5
    f.val = vals.copy()
    assert np.array_equal(jv.apply_preconditioner(f, r), expected_apply(f, vals, r))


def test_sibling_copy_does_not_leak(rng):
    """Two IluFactors over one pattern share the device buffer: each call
    must see its own values."""
    a, f = make()
    g = f.copy()
    jv.factor_serial(f)
    g.val[:] = g.val * 1.5
    jv.factor_serial(g)
    fv, gv = f.val.copy(), g.val.copy()
    r = rng.uniform(-1, 1, a.n)
    for _ in range(2):
        assert np.array_equal(jv.apply_preconditioner(f, r), expected_apply(f, fv, r))
        assert np.array_equal(jv.apply_preconditioner(g, r), expected_apply(g, gv, r))


def test_zero_pivot_leaves_host_state_authoritative(rng):
    a = jv.CsrMatrix.from_dense(np.array([[1.0, 1.0, 0.0], [1.0, 1.0, 1.0], [0.0, 1.0, 1.0]]))
    f = jv.assemble_factors(a, a.pattern, jv.Permutation.identity(3))
    with pytest.raises(jv.ZeroPivotError):
        jv.factor_serial(f)
    vals = f.val.copy()
    b = np.array([1.0, 2.0, 3.0])
    rs, col = f.pattern.row_start.astype(np.int64), f.pattern.col.astype(np.int64)
    assert np.array_equal(jv.solve_serial(f, b, "forward"), oracle.solve_forward(rs, col, vals, b))


@pytest.mark.parametrize("runs", [[(0, 100), (200, 330)], [(5, 6), (7, 8), (9, 300), (400, 576)]])
def test_factor_parallel_upper_row_runs(runs):
    a, f = make()
    rows = np.concatenate([np.arange(lo, hi) for lo, hi in runs])
    sched = types.SimpleNamespace(order=rows[::-1].copy())   # any order: only the set matters
    rs = f.pattern.row_start.astype(np.int64)
    col = f.pattern.col.astype(np.int64)
    diag = f.diag_pos.astype(np.int64)
    want = f.val.copy()
    lib = oracle.lib()
    norms = np.zeros(a.n)
    for lo, hi in runs:
        lib.or_factor_rows(oracle._p(rs), oracle._p(col), oracle._p(want), oracle._p(diag),
                           oracle._p(norms), 0.0, 0, lo, hi, 0, a.n)
    jv.factor_parallel_upper(f, sched)
    assert np.array_equal(f.val, want)


def test_spmv_keeps_the_matrix_resident(uploads, rng):
    """The reference's Krylov loop calls spmv(a, p) per iteration
    (krylov.py:52-151): the matrix is uploaded once, and again only after
    the caller could have changed it."""
    a = jv.poisson2d(24)
    rs, col, val = a.row_start.astype(np.int64), a.col.astype(np.int64), a.val.copy()
    uploads.clear()
    xs = [rng.uniform(-1, 1, a.n) for _ in range(4)]
    for x in xs:
        assert np.array_equal(jv.spmv(a, x), oracle.spmv(rs, col, val, x))
    assert len(uploads) == 1, uploads           # (the a.val read above came first)
    a.val[:] *= 2.0                             # in-place edit through the attribute
    assert np.array_equal(jv.spmv(a, xs[0]), oracle.spmv(rs, col, 2.0 * val, xs[0]))
    assert len(uploads) == 2
    alias = a.val                               # a kept alias: never trusted
    jv.spmv(a, xs[0])
    alias[0] = 7.0
    val2 = 2.0 * val
    val2[0] = 7.0
    assert np.array_equal(jv.spmv(a, xs[1]), oracle.spmv(rs, col, val2, xs[1]))
    a.val = val.copy()                          # rebinding
    del alias
    assert np.array_equal(jv.spmv(a, xs[2]), oracle.spmv(rs, col, val, xs[2]))
    n_up = len(uploads)
    assert np.array_equal(jv.spmv(a, xs[3]), oracle.spmv(rs, col, val, xs[3]))
    assert len(uploads) == n_up


def test_long_vectors_come_back_in_pinned_memory(rng):
    """Results of the drop-in solves of at least 2^17 entries are written by
    one DMA into page-locked memory; the caller owns the array."""
    from paper_1812_06160_b200 import workloads as W

    a = W.laplace7(52)                           # 140,608 rows
    f = jv.assemble_factors(a, jv.ilu0_pattern(a.pattern), jv.Permutation.identity(a.n))
    jv.factor_serial(f)
    vals = f.val.copy()
    r = rng.uniform(-1, 1, a.n)
    z = jv.apply_preconditioner(f, r)
    assert z.flags.writeable and z.dtype == np.float64 and z.shape == (a.n,)
    assert np.array_equal(z, expected_apply(f, vals, r))
    keep = z.copy()
    z2 = jv.apply_preconditioner(f, 2.0 * r)     # a second result must not alias the first
    assert np.array_equal(z, keep) and not np.shares_memory(z, z2)
    with pytest.raises(ValueError):
        jv.apply_preconditioner(f, r[:-1])
