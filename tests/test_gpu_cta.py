"""The single-CTA level-synchronous kernels (csrc/cta.cu): factor and both
sweeps bitwise equal to the reference's golden vectors and to the pinned
oracle, with values in shared memory (small) and in L2 (larger), tau drops
and MILU; zero pivots report the smallest row."""

import numpy as np
import pytest

import oracle
from conftest import golden_names

pytestmark = pytest.mark.gpu

jv = pytest.importorskip("paper_1812_06160_b200")
from paper_1812_06160_b200 import device as dv  # noqa: E402
from paper_1812_06160_b200.plan import build_plan  # noqa: E402

CUTS = {"poisson2d_16_cut2": 2, "rdd150_tau_milu_cut3": 3, "rdd200_cut4": 4}


@pytest.mark.parametrize("name", golden_names())
def test_cta_matches_reference(golden, name):
    g = golden.case(name)
    n = g["a_rs"].size - 1
    a = jv.CsrMatrix(n, g["a_rs"], g["a_col"], g["a_val"])
    plan = build_plan(a, k=int(g["k"]), tau=float(g["tau"]), milu=bool(g["milu"]),
                      cut=CUTS.get(name))
    ilu = plan.ilu
    ilu._factor_cta(True)
    bad = dv.read_row_slot(ilu.err)
    assert bad == int(g["bad"])
    if bad >= 0:
        return
    assert np.array_equal(ilu.host_val(), g["fval"])
    b = dv.f64(g["b"])
    y, x = dv.empty_f64(n), dv.empty_f64(n)
    ilu._solve_cta(0, b, y)
    ilu._solve_cta(1, y, x)
    assert np.array_equal(dv.host_f64(y, n), g["y"])
    assert np.array_equal(dv.host_f64(x, n), g["x"])
    ilu._solve_cta(0, b, b)          # in place
    assert np.array_equal(dv.host_f64(b, n), g["y"])


@pytest.mark.parametrize("side", [30, 120, 170])
@pytest.mark.parametrize("k,tau,milu", [(0, 0.0, False), (1, 0.0, False), (1, 0.03, True)])
def test_cta_against_oracle(side, k, tau, milu):
    """side 30: everything in shared memory; 120: values in L2, vector in
    shared memory; 170: both in L2."""
    a = jv.convdiff2d(side, seed=side)
    plan = build_plan(a, k=k, tau=tau, milu=milu)
    ilu = plan.ilu
    n = ilu.n
    rs = dv.host_i64(ilu.row_start, n + 1)
    col = dv.host_i64(ilu.col, ilu.nnz)
    diag = dv.host_i64(ilu.diag_pos, n)
    want, wbad = oracle.factor_serial(rs, col, dv.host_f64(plan.assembled, ilu.nnz), diag, tau,
                                      milu)
    ilu._factor_cta(True)
    assert dv.read_row_slot(ilu.err) == wbad == -1
    got = ilu.host_val()
    assert np.array_equal(got, want)
    b = np.random.default_rng(side).uniform(-1, 1, n)
    bd, y, x = dv.f64(b), dv.empty_f64(n), dv.empty_f64(n)
    ilu._solve_cta(0, bd, y)
    ilu._solve_cta(1, y, x)
    yo = oracle.solve_forward(rs, col, want, b)
    xo, _ = oracle.solve_backward(rs, col, want, diag, yo)
    assert np.array_equal(dv.host_f64(y, n), yo)
    assert np.array_equal(dv.host_f64(x, n), xo)


def test_cta_zero_pivot_smallest_row():
    n = 900
    d = np.zeros((n, n))
    for i in range(n):
        d[i, i] = 4.0
        if i + 1 < n:
            d[i, i + 1] = d[i + 1, i] = -1.0
    for r in (611, 233, 402):
        d[r, :] = 0.0
        d[:, r] = 0.0
    a = jv.CsrMatrix.from_dense(d, keep=(d != 0.0) | np.eye(n, dtype=bool))
    plan = build_plan(a)
    ilu = plan.ilu
    ilu._factor_cta(True)
    perm = dv.host_i64(plan.perm, n)
    inv = np.argsort(perm)
    assert dv.read_row_slot(ilu.err) == min(inv[[611, 233, 402]])


def test_cta_is_an_autotune_candidate_and_picked_for_c1():
    a = jv.poisson2d(64)
    plan = build_plan(a)
    ilu = plan.ilu
    ilu.region_mode = "auto"
    assert ilu.factor() == -1
    want = ilu.host_val()
    for sw in ("factor", "fwd", "bwd"):
        ilu._region_for(sw)
    for _ in range(3):
        plan.reset_values()
        ilu._factor_cta(True)
        assert np.array_equal(ilu.host_val(), want)
