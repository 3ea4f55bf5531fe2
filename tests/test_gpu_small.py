"""jv_solve_small (one thread block, the whole sweep in shared memory)
against the golden cases and the oracle, bitwise; it is a candidate of the
solves' one-time path timing and wins on config 1."""
import os
import sys

import numpy as np
import pytest

import oracle

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
pytestmark = pytest.mark.gpu

import paper_1812_06160_b200 as jv  # noqa: E402
from paper_1812_06160_b200 import device as dv  # noqa: E402
from paper_1812_06160_b200 import workloads as W  # noqa: E402
from paper_1812_06160_b200.plan import build_plan  # noqa: E402


def _check(plan, seed=0):
    ilu = plan.ilu
    n = ilu.n
    assert ilu.factor() == -1
    rs = dv.host_i64(ilu.row_start, n + 1)
    col = dv.host_i64(ilu.col, ilu.nnz)
    diag = dv.host_i64(ilu.diag_pos, n)
    val = ilu.host_val()
    b = np.random.default_rng(seed).uniform(-1.0, 1.0, n)
    yo = oracle.solve_forward(rs, col, val, b)
    xo, _ = oracle.solve_backward(rs, col, val, diag, yo)
    assert ilu._small_plan(0) is not None and ilu._small_plan(1) is not None
    bd, y, x = dv.f64(b), dv.empty_f64(n), dv.empty_f64(n)
    ilu._solve_small(0, bd, y)
    ilu._solve_small(1, y, x)
    assert np.array_equal(dv.host_f64(y, n), yo)
    assert np.array_equal(dv.host_f64(x, n), xo)
    ilu._solve_small(0, bd, bd)            # in place
    ilu._solve_small(1, bd, bd)
    assert np.array_equal(dv.host_f64(bd, n), xo)


@pytest.mark.parametrize("case", ["poisson2d_64", "laplace7_12_ilu1", "convdiff3d_10_ilu2_tau",
                                  "rmat_10"])
def test_small_solves_bitwise(case):
    a, kw = {"poisson2d_64": (lambda: jv.poisson2d(64), {}),
             "laplace7_12_ilu1": (lambda: W.laplace7(12), dict(k=1)),
             "convdiff3d_10_ilu2_tau": (lambda: W.convdiff3d(10), dict(k=2, tau=1e-3)),
             "rmat_10": (lambda: W.rmat(10, 3), {})}[case]
    _check(build_plan(a(), **kw))


def test_too_large_systems_have_no_small_plan():
    plan = build_plan(W.laplace7(40))          # 64,000 rows
    assert plan.ilu._small_plan(0) is None and plan.ilu._small_plan(1) is None


def test_small_is_an_autotune_candidate_on_config_1():
    plan = build_plan(jv.poisson2d(64))
    ilu = plan.ilu
    ilu.region_mode = "auto"
    assert ilu.factor() == -1
    n = ilu.n
    b = dv.f64(np.random.default_rng(1).uniform(-1.0, 1.0, n))
    y, x = dv.empty_f64(n), dv.empty_f64(n)
    ilu.solve_async(0, b, y)
    ilu.solve_async(1, y, x)
    for sw in ("fwd", "bwd"):
        assert len(ilu.autotune_ms[sw]) >= 3      # tickets, region(s), ..., small
    rs = dv.host_i64(ilu.row_start, n + 1)
    col = dv.host_i64(ilu.col, ilu.nnz)
    diag = dv.host_i64(ilu.diag_pos, n)
    yo = oracle.solve_forward(rs, col, ilu.host_val(), dv.host_f64(b, n))
    xo, _ = oracle.solve_backward(rs, col, ilu.host_val(), diag, yo)
    assert np.array_equal(dv.host_f64(x, n), xo)
