"""The two-stage lower tail (csrc/tail.cu): stage 1
eliminates each tail row's upper-stage pivots with the segmented warp
kernel, stage 2 factors the compact corner; bitwise equal to the reference
factor_serial (golden vectors) and to the pinned oracle on random matrices
with forced cuts, ILU(1) fill, tau drops and MILU."""

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
def test_device_two_stage_matches_reference(golden, name):
    g = golden.case(name)
    n = g["a_rs"].size - 1
    a = jv.CsrMatrix(n, g["a_rs"], g["a_col"], g["a_val"])
    plan = build_plan(a, k=int(g["k"]), tau=float(g["tau"]), milu=bool(g["milu"]),
                      cut=CUTS.get(name))
    ilu = plan.ilu
    if plan.n_upper >= n:
        pytest.skip("no lower tail")
    if plan.n_upper:
        ilu._factor_tickets(0, plan.n_upper, 0, True)
    bad = ilu.factor_tail(plan.n_upper)
    assert bad == int(g["bad"])
    if bad < 0:
        assert np.array_equal(ilu.host_val(), g["fval"])
    dv.check_hang()


def _random_case(seed, k, tau, milu, cut_frac):
    a = jv.random_diag_dominant(300 + 41 * seed, row_nnz=4 + seed % 4, seed=100 + seed,
                                symmetric_pattern=bool(seed % 2))
    # forced cut: the last `cut_frac` of the levels form the tail
    pre = build_plan(a, k=k)
    cut = max(0, int(pre.nlev * (1.0 - cut_frac)))
    plan = build_plan(a, k=k, tau=tau, milu=milu, cut=cut)
    return plan


@pytest.mark.parametrize("seed", range(6))
@pytest.mark.parametrize("k,tau,milu", [(0, 0.0, False), (1, 0.0, False), (1, 0.05, False),
                                        (0, 0.05, True), (1, 0.02, True), (0, 0.0, True)])
@pytest.mark.parametrize("cut_frac", [0.3, 1.0])
def test_tail_random_against_oracle(seed, k, tau, milu, cut_frac):
    plan = _random_case(seed, k, tau, milu, cut_frac)
    ilu = plan.ilu
    n = ilu.n
    rs = dv.host_i64(ilu.row_start, n + 1)
    col = dv.host_i64(ilu.col, ilu.nnz)
    diag = dv.host_i64(ilu.diag_pos, n)
    assembled = dv.host_f64(plan.assembled, ilu.nnz)
    want, wbad = oracle.factor_serial(rs, col, assembled, diag, tau, milu)
    if wbad >= 0:
        pytest.skip("zero pivot in the random case")
    ilu.factor_two_stage_async(plan.n_upper)
    got = ilu.host_val()
    assert dv.read_row_slot(ilu.tail_plan(plan.n_upper).corner.err) < 0
    assert np.array_equal(got, want)
    tp = ilu.tail_plan(plan.n_upper)
    assert tp.nt == n - plan.n_upper
    dv.check_hang()


def test_tail_plan_groups_are_independent():
    """Every group of a tail row receives no update from its own pivots
    (the precondition of the parallel DIVIDE)."""
    a = jv.random_diag_dominant(500, row_nnz=7, seed=3)
    plan = build_plan(a, k=1, cut=1)
    tp = plan.ilu.tail_plan(plan.n_upper)
    assert tp.nt == a.n - plan.n_upper and tp.ngroups > 0
    assert tp.nsegs <= tp.nops


def test_two_stage_is_an_autotune_candidate():
    a = jv.random_diag_dominant(400, row_nnz=6, seed=9)
    plan = build_plan(a, cut=2)
    ilu = plan.ilu
    ilu.region_mode = "auto"
    ilu.factor()
    want = ilu.host_val()
    for _ in range(3):
        plan.reset_values()
        ilu.factor_two_stage_async(plan.n_upper)
        assert np.array_equal(ilu.host_val(), want)
