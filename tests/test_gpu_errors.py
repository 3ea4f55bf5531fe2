"""The reference's error-path cases, run through the device API
(`-m gpu`): missing diagonals, uncovered / mismatched patterns, the `which`
check, zero pivots in the factorization (smallest row, state after the
error) and in the backward sweep (minimum row, every path), the forward
sweep ignoring the stored diagonal, schedule size mismatches.

Reference: pkg/tests/test_symbolic.py:23-28,99-116,
pkg/tests/test_trisolve.py:34,146-176, pkg/tests/test_factor.py (zero
pivots), pkg/tests/test_lower.py (two-stage zero pivots)."""

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

jv = pytest.importorskip("paper_1812_06160_b200")
from paper_1812_06160_b200.ordering import LOWER_A_PLUS_AT  # noqa: E402
from paper_1812_06160_b200.trisolve import BACKWARD, FORWARD  # noqa: E402


def factored(a, k=0):
    pattern, _ = jv.iluk_pattern(a.pattern, k)
    f = jv.assemble_factors(a, pattern, jv.Permutation.identity(a.n))
    jv.factor_serial(f)
    return f


# ---- symbolic (test_symbolic.py) ------------------------------------------

def test_ilu0_missing_diagonal_reports_row():
    a = jv.CsrMatrix.from_coo(3, [0, 1, 2], [0, 1, 0], [1.0, 1.0, 1.0])
    with pytest.raises(jv.MissingDiagonalError) as exc:
        jv.ilu0_pattern(a.pattern)
    assert exc.value.row == 2


@pytest.mark.parametrize("k", [1, 2])
def test_iluk_missing_diagonal_reports_first_row(k):
    a = jv.CsrMatrix.from_coo(4, [0, 1, 1, 2, 3], [0, 0, 2, 2, 1], [1.0] * 5)
    with pytest.raises(jv.MissingDiagonalError) as exc:
        jv.iluk_pattern(a.pattern, k)
    assert exc.value.row == 1


def test_assemble_rejects_uncovered_pattern():
    a = jv.tridiag(4)
    small = jv.CsrMatrix.from_dense(np.eye(4)).pattern
    with pytest.raises(jv.MatrixFormatError):
        jv.assemble_factors(a, small, jv.Permutation.identity(4))


def test_assemble_rejects_missing_diagonal():
    a = jv.CsrMatrix.from_coo(2, [0, 0, 1], [0, 1, 0], [1.0, 2.0, 3.0])
    with pytest.raises(jv.MissingDiagonalError) as exc:
        jv.assemble_factors(a, a.pattern, jv.Permutation.identity(2))
    assert exc.value.row == 1


def test_assemble_size_mismatch():
    a = jv.tridiag(4)
    with pytest.raises(jv.MatrixFormatError):
        jv.assemble_factors(a, jv.tridiag(5).pattern, jv.Permutation.identity(4))


# ---- factorization zero pivots (factor.py:37-63) ---------------------------

def test_factor_zero_pivot_smallest_row_and_state():
    """ZeroPivotError(smallest row); rows after it keep their input values,
    as the reference's serial kernel stops there (_kernels.py:197-204)."""
    a = jv.CsrMatrix.from_dense([[1.0, 1.0, 0.0, 0.0], [1.0, 1.0, 1.0, 0.0],
                                 [0.0, 1.0, 2.0, 1.0], [0.0, 0.0, 1.0, 2.0]])
    pat, _ = jv.iluk_pattern(a.pattern, 0)
    f = jv.assemble_factors(a, pat, jv.Permutation.identity(4))
    before = f.val.copy()
    want, bad = oracle.factor_serial(pat.row_start, pat.col, before, f.diag_pos)
    assert bad == 1
    with pytest.raises(jv.ZeroPivotError) as exc:
        jv.factor_serial(f)
    assert exc.value.row == 1
    rs = pat.row_start
    # rows up to the failing one: the oracle's values; later rows: input
    assert np.array_equal(f.val[:rs[2]], want[:rs[2]])
    assert np.array_equal(f.val[rs[2]:], before[rs[2]:])


def test_factor_zero_pivot_many_rows_reports_min():
    """Several zero pivots in independent rows: the smallest row wins
    regardless of which warp finds its zero first (factor.py:61-63)."""
    n = 300
    d = np.zeros((n, n))
    for i in range(n):
        d[i, i] = 4.0
        if i + 1 < n:
            d[i, i + 1] = d[i + 1, i] = -1.0
    for r in (251, 73, 140):    # decoupled rows with a stored zero diagonal
        d[r, :] = 0.0
        d[:, r] = 0.0
    keep = (d != 0.0) | np.eye(n, dtype=bool)
    a = jv.CsrMatrix.from_dense(d, keep=keep)
    pat, _ = jv.iluk_pattern(a.pattern, 0)
    f = jv.assemble_factors(a, pat, jv.Permutation.identity(n))
    _, bad = oracle.factor_serial(pat.row_start, pat.col, f.val.copy(), f.diag_pos)
    assert bad == 73
    with pytest.raises(jv.ZeroPivotError) as exc:
        jv.factor_serial(f)
    assert exc.value.row == 73


def _chain_with_tail_zero_pivot(n, zrow):
    """Tridiagonal chain whose row `zrow` eliminates to exactly 0."""
    d = np.zeros((n, n))
    for i in range(n):
        d[i, i] = 4.0
        if i + 1 < n:
            d[i, i + 1] = d[i + 1, i] = -1.0
    a = jv.CsrMatrix.from_dense(d)
    pat, _ = jv.iluk_pattern(a.pattern, 0)
    f = jv.assemble_factors(a, pat, jv.Permutation.identity(n))
    fv, _ = oracle.factor_serial(pat.row_start, pat.col, f.val.copy(), f.diag_pos)
    u = fv[f.diag_pos[zrow - 1]]
    l = np.float64(-1.0) / u
    d[zrow, zrow] = l * np.float64(-1.0)     # diag - l*u_{zrow-1,zrow} == 0 exactly
    return jv.CsrMatrix.from_dense(d)


@pytest.mark.parametrize("method", ["er", "sr"])
def test_two_stage_zero_pivot_in_tail_state(method):
    """A zero pivot in the lower tail: the tail stage raises that row and the
    later tail rows keep their post-upper-stage values, as the reference's
    corner kernel stops there (lower.py:261-270)."""
    n = 64
    a = _chain_with_tail_zero_pivot(n, n - 3)
    src = jv.lower_pattern(jv.symmetrize_pattern(a.pattern))
    sched = jv.compute_levels(src, LOWER_A_PLUS_AT)
    levels = sched.levels
    cut = len(levels) - 6
    part = jv.StagePartition([r.copy() for r in levels[:cut]],
                             np.concatenate(levels[cut:]), cut)
    perm = jv.build_level_permutation(part)
    pa = jv.permute_symmetric(a, perm)
    pat, _ = jv.iluk_pattern(pa.pattern, 0)
    f = jv.assemble_factors(a, pat, perm)
    ser = f.copy()
    with pytest.raises(jv.ZeroPivotError) as e0:
        jv.factor_serial(ser)
    assert e0.value.row == n - 3
    sync = jv.build_sync_schedule(part, f.pattern, 2)
    jv.factor_parallel_upper(f, sync)
    after_upper = f.val.copy()
    with pytest.raises(jv.ZeroPivotError) as e1:
        if method == "er":
            jv.factor_er(f, part, nthreads=2)
        else:
            jv.factor_sr(f, jv.build_tiles(f, part), nthreads=2)
    assert e1.value.row == n - 3
    rs = pat.row_start
    bad = n - 3
    assert np.array_equal(f.val[:rs[bad + 1]], ser.val[:rs[bad + 1]])
    assert np.array_equal(f.val[rs[bad + 1]:], after_upper[rs[bad + 1]:])


# ---- solves (test_trisolve.py) --------------------------------------------

def test_which_is_checked():
    f = factored(jv.tridiag(4))
    with pytest.raises(ValueError):
        jv.solve_serial(f, np.ones(4), "sideways")
    with pytest.raises(ValueError):
        jv.solve_ls(f, np.ones(4), None, "up")


def zeroed_diag_factors():
    f = factored(jv.tridiag(8))
    f.val[f.diag_pos[5]] = 0.0
    f.val[f.diag_pos[3]] = 0.0
    return f


def test_backward_zero_diagonal_raises_min_row_every_path():
    f = zeroed_diag_factors()
    b = np.ones(8)
    with pytest.raises(jv.ZeroPivotError) as e1:
        jv.solve_serial(f, b, BACKWARD)
    assert e1.value.row == 3
    setup = jv.build_solve_setup(f, "csrls", 2)
    with pytest.raises(jv.ZeroPivotError) as e2:
        jv.solve_baseline_csrls(f, b, setup.bwd_levels, 2, BACKWARD)
    assert e2.value.row == 3
    setup = jv.build_solve_setup(f, "ls", 2)
    with pytest.raises(jv.ZeroPivotError) as e3:
        jv.solve_ls(f, b, setup.bwd_sync, BACKWARD)
    assert e3.value.row == 3
    with pytest.raises(jv.ZeroPivotError) as e4:
        jv.apply_preconditioner(f, b)
    assert e4.value.row == 3


def test_forward_ignores_stored_diagonal():
    f = zeroed_diag_factors()
    y = jv.solve_serial(f, np.ones(8), FORWARD)
    assert np.all(np.isfinite(y))
    want = oracle.solve_forward(f.pattern.row_start, f.pattern.col, f.val, np.ones(8))
    assert np.array_equal(y, want)


def test_schedule_size_mismatch_rejected():
    f = factored(jv.tridiag(8))
    small = jv.compute_levels(jv.lower_pattern(jv.tridiag(4).pattern))
    with pytest.raises(jv.ConfigurationError):
        jv.solve_baseline_csrls(f, np.ones(8), small, 2, FORWARD)
    small_sync = jv.build_triangle_schedule(jv.tridiag(4).pattern, 2, FORWARD)
    with pytest.raises(jv.ConfigurationError):
        jv.solve_ls(f, np.ones(8), small_sync, FORWARD)


def test_preconditioner_keeps_its_own_values():
    """A preconditioner built from one factor copy is not affected by later
    uploads of sibling copies over the same pattern (advisor finding)."""
    a = jv.poisson2d(12)
    f = factored(a)
    pre = jv.ilu_preconditioner(f)
    r = np.linspace(-1.0, 1.0, a.n)
    z0 = pre(r)
    g = f.copy()
    g.val[:] = 1.0 + np.arange(g.val.size) % 3     # a different factor on the same pattern
    jv.solve_serial(g, r, FORWARD)                 # uploads g's values
    assert np.array_equal(pre(r), z0)
    assert np.array_equal(z0, jv.apply_preconditioner(f, r))
