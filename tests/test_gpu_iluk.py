"""Device ILU(k >= 2) symbolic factorization (jv_iluk_round, k rounds of the
level-of-fill closure) against the row-by-row algorithm (symbolic.py:86-138;
libjv's host C++ restatement, itself pinned by the golden ILU(2) cases) and
against the pinned oracle's C restatement: patterns and fill levels equal."""
import os
import sys

import numpy as np
import pytest

import oracle

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
pytestmark = pytest.mark.gpu

import paper_1812_06160_b200 as jv  # noqa: E402
from paper_1812_06160_b200 import symbolic as sym  # noqa: E402
from paper_1812_06160_b200 import workloads as W  # noqa: E402
from paper_1812_06160_b200.csr import SparsityPattern  # noqa: E402


def _random_pattern(rng, n, per_row):
    rows = np.repeat(np.arange(n), per_row)
    cols = rng.integers(0, n, rows.size)
    rows = np.concatenate((rows, np.arange(n)))      # full diagonal
    cols = np.concatenate((cols, np.arange(n)))
    key = np.unique(rows * n + cols)
    r, c = key // n, key % n
    rs = np.zeros(n + 1, dtype=np.int64)
    np.add.at(rs, r + 1, 1)
    return SparsityPattern(n, np.cumsum(rs), c)


@pytest.mark.parametrize("k", [2, 3, 4, 7])
@pytest.mark.parametrize("case", ["random_sparse", "random_denser", "laplace7", "convdiff3d"])
def test_device_rounds_equal_row_by_row(case, k):
    rng = np.random.default_rng(17)
    pat = {"random_sparse": lambda: _random_pattern(rng, 400, 2),
           "random_denser": lambda: _random_pattern(rng, 150, 5),
           "laplace7": lambda: W.laplace7(9).pattern,
           "convdiff3d": lambda: W.convdiff3d(8).pattern}[case]()
    got, glev = jv.iluk_pattern(pat, k)               # device rounds
    want, wlev = sym._iluk_host(pat, k)               # row-by-row
    assert np.array_equal(got.row_start, want.row_start)
    assert np.array_equal(got.col, want.col)
    assert np.array_equal(glev.level, wlev.level)
    assert glev.level.max() <= k


def test_device_rounds_equal_oracle_numpy():
    rng = np.random.default_rng(3)
    pat = _random_pattern(rng, 120, 3)
    for k in (2, 3):
        got, glev = jv.iluk_pattern(pat, k)
        rs, col, lev = oracle.iluk_pattern(pat.row_start, pat.col, k)   # pinned C restatement
        assert np.array_equal(got.row_start, rs) and np.array_equal(got.col, col)
        assert np.array_equal(glev.level, lev)


def test_plan_uses_device_rounds_and_factors_bitwise():
    """ILU(2, tau) through the all-in-HBM plan: pattern from the device rounds,
    factor values bitwise the oracle's on that pattern."""
    a = W.convdiff3d(10)
    from paper_1812_06160_b200 import device as dv
    from paper_1812_06160_b200.plan import build_plan

    plan = build_plan(a, k=2, tau=1e-3)
    ilu = plan.ilu
    n = a.n
    rs = dv.host_i64(ilu.row_start, n + 1)
    col = dv.host_i64(ilu.col, ilu.nnz)
    diag = dv.host_i64(ilu.diag_pos, n)
    assembled = ilu.host_val()
    assert ilu.factor() == -1
    want, bad = oracle.factor_serial(rs, col, assembled, diag, tau=1e-3)
    assert bad == -1 and np.array_equal(ilu.host_val(), want)
