"""GPU parity of the CTA-resident region kernels (csrc/region.cu): forced on,
the factorization (stencil-class matrices) and both solves must equal the
CPU oracle bit for bit, and the ticket kernels too; zero pivots are reported
as the smallest row, as the reference does (factor.py:61-63)."""

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

jv = pytest.importorskip("paper_1812_06160_b200")
from paper_1812_06160_b200 import device as dv  # noqa: E402
from paper_1812_06160_b200 import workloads as W  # noqa: E402


def _case(name):
    return {
        "poisson2d_48": (W.poisson2d(48), 0, 0.0),
        "laplace7_20": (W.laplace7(20, 1), 0, 0.0),
        "laplace7_20_tau": (W.laplace7(20, 2), 0, 0.05),
        "convdiff3d_12_ilu1": (W.convdiff3d(12, 3), 1, 1e-3),
        "stencil27_12": (W.stencil27(12, 4), 0, 0.0),
        "random_dd_5000": (W.random_diag_dominant(5000, 7, seed=9), 0, 0.0),
    }[name]


NAMES = ["poisson2d_48", "laplace7_20", "laplace7_20_tau", "convdiff3d_12_ilu1",
         "stencil27_12", "random_dd_5000"]


def _front(a, k, tau):
    fe = oracle.front_end(a.n, a.row_start, a.col, a.val, k=k, tau=tau)
    return fe["row_start"], fe["col"], fe["diag"], fe["val"]


@pytest.mark.parametrize("name", NAMES)
@pytest.mark.parametrize("mode", ["on", "on-single", "off", "auto"])
def test_region_paths_bitwise(name, mode):
    """on: one region per SM (cross-region mailboxes); on-single: the whole
    matrix in one CTA; off: ticket kernels; auto: the faster per sweep."""
    a, k, tau = _case(name)
    rs, col, diag, val = _front(a, k, tau)
    n = diag.size
    want, bad = oracle.factor_serial(rs, col, val.copy(), diag, tau, False)
    assert bad < 0
    d = dv.DevIlu.from_host(n, rs, col, diag, val, tau=tau)
    d.region_single_max = n if mode == "on-single" else 0
    d.region_mode = "on" if mode.startswith("on") else mode
    if mode == "on-single":
        assert d.regions()[0] == 1
    if mode == "on":
        assert d.region_stream("fwd") is not None and d.region_stream("bwd") is not None
        stencil = name.startswith(("poisson", "laplace"))
        assert (d.region_stream("factor") is not None) == stencil
    assert d.factor() == -1
    assert np.array_equal(d.host_val(), want)
    b = np.random.default_rng(1).uniform(-1, 1, n)
    y = dv.empty_f64(n)
    x = dv.empty_f64(n)
    for rep in range(2):   # mailbox epochs advance between calls
        d.solve_async(0, dv.f64(b), y)
        d.solve_async(1, y, x)
        yo = oracle.solve_forward(rs, col, want, b)
        xo, _ = oracle.solve_backward(rs, col, want, diag, yo)
        assert np.array_equal(dv.host_f64(y, n), yo)
        assert np.array_equal(dv.host_f64(x, n), xo)
    dv.check_hang()


def test_region_factor_zero_pivot_smallest_row():
    """A zero pivot in the middle of a stencil matrix: the region factor
    reports the smallest bad row, like the reference."""
    a = W.poisson2d(40)
    rs, col, diag, val = _front(a, 0, 0.0)
    n = diag.size
    val = val.copy()
    # make two rows singular after elimination: zero their diagonal and
    # their strictly-lower entries
    for r in (900, 1300):
        val[rs[r]:diag[r] + 1] = 0.0
    want, bad = oracle.factor_serial(rs, col, val.copy(), diag, 0.0, False)
    assert bad == 900
    d = dv.DevIlu.from_host(n, rs, col, diag, val)
    d.region_single_max = 0
    d.region_mode = "on"
    assert d.region_stream("factor") is not None
    assert d.factor() == 900
    got = d.host_val()
    upto = rs[bad + 1]
    assert np.array_equal(got[:upto], want[:upto])


def test_region_many_epochs():
    """Repeated launches (epochs) on one plan stay bitwise and never hang."""
    a = W.laplace7(16, 5)
    rs, col, diag, val = _front(a, 0, 0.0)
    n = diag.size
    want, _ = oracle.factor_serial(rs, col, val.copy(), diag, 0.0, False)
    d = dv.DevIlu.from_host(n, rs, col, diag, val)
    d.region_single_max = 0
    d.region_mode = "on"
    for _ in range(20):
        dv.upload_f64(d.val, val)
        assert d.factor() == -1
    assert np.array_equal(d.host_val(), want)
    dv.check_hang()


@pytest.mark.parametrize("k", [0, 1])
def test_csrls_baseline_bitwise(k):
    """The paper's CSR-LS baseline (one launch per level, CUDA graph) gives
    the reference's bits, like every other solve path."""
    from paper_1812_06160_b200.ordering import LOWER_A_PLUS_AT
    from paper_1812_06160_b200.trisolve import BACKWARD, FORWARD
    a = W.convdiff3d(8, 2) if k else W.laplace7(12, 4)
    src = jv.lower_pattern(jv.symmetrize_pattern(a.pattern))
    sched = jv.compute_levels(src, LOWER_A_PLUS_AT)
    part = jv.partition_stages(sched, np.diff(a.row_start))
    perm = jv.build_level_permutation(part)
    permuted = jv.permute_symmetric(a, perm)
    pattern, _ = jv.iluk_pattern(permuted.pattern, k)
    f = jv.assemble_factors(a, pattern, perm)
    jv.factor_serial(f)
    b = np.random.default_rng(3).uniform(-1, 1, a.n)
    rs, col, val, dg = f.pattern.row_start, f.pattern.col, f.val, f.diag_pos
    yo = oracle.solve_forward(rs, col, val, b)
    xo, _ = oracle.solve_backward(rs, col, val, dg, yo)
    for rep in range(2):
        y = jv.solve_baseline_csrls(f, b, sched, 8, FORWARD)
        x = jv.solve_baseline_csrls(f, y, sched, 8, BACKWARD)
        assert np.array_equal(y, yo) and np.array_equal(x, xo)


@pytest.mark.parametrize("mode", ["auto", "on"])
def test_zero_pivot_any_path(mode):
    """Whatever path the autotune picks, the smallest zero-pivot row."""
    a = W.laplace7(14, 2)
    rs, col, diag, val = _front(a, 0, 0.0)
    val = val.copy()
    for r in (700, 1500):
        val[rs[r]:diag[r] + 1] = 0.0
    want, bad = oracle.factor_serial(rs, col, val.copy(), diag, 0.0, False)
    d = dv.DevIlu.from_host(diag.size, rs, col, diag, val)
    d.region_single_max = 0
    d.region_mode = mode
    assert d.factor() == bad == 700
    upto = rs[bad + 1]
    assert np.array_equal(d.host_val()[:upto], want[:upto])


def test_solves_follow_refactorization():
    """New values -> factor -> the region solves see the new factors (the
    wave-ordered value copies are refreshed per factorization)."""
    a = W.laplace7(12, 6)
    rs, col, diag, val = _front(a, 0, 0.0)
    n = diag.size
    d = dv.DevIlu.from_host(n, rs, col, diag, val)
    d.region_single_max = 0
    d.region_mode = "on"
    b = np.random.default_rng(2).uniform(-1, 1, n)
    y, x = dv.empty_f64(n), dv.empty_f64(n)
    for scale in (1.0, 2.0, 0.5):
        v = val * scale
        dv.upload_f64(d.val, v)
        d.values_changed()
        assert d.factor() == -1
        want, _ = oracle.factor_serial(rs, col, v.copy(), diag, 0.0, False)
        d.solve_async(0, dv.f64(b), y)
        d.solve_async(1, y, x)
        yo = oracle.solve_forward(rs, col, want, b)
        xo, _ = oracle.solve_backward(rs, col, want, diag, yo)
        assert np.array_equal(dv.host_f64(x, n), xo)


@pytest.mark.parametrize("mode", ["on", "auto"])
def test_refactor_new_values_region_packs(mode):
    """Refactorization with new values of the same pattern: the value packs
    (the backward one refreshed on a side stream during the forward sweep)
    may never be stale.  Checked bitwise against the oracle for each set of
    values."""
    a = W.laplace7(18, 5)
    rs, col, diag, val0 = _front(a, 0, 0.0)
    n = diag.size
    d = dv.DevIlu.from_host(n, rs, col, diag, val0, tau=0.0)
    d.region_mode = mode
    src = dv.f64(val0)
    b = np.random.default_rng(3).uniform(-1, 1, n)
    bd = dv.f64(b)
    y, x = dv.empty_f64(n), dv.empty_f64(n)
    rng = np.random.default_rng(4)
    for rep in range(4):
        v = val0 * rng.uniform(0.5, 1.5, val0.size)
        v[diag] = np.abs(val0[diag]) * (2.0 + rep)
        src.copy_(dv.f64(v))
        d.load_values(src)
        d.factor_async()
        d.solve_async(0, bd, y)
        d.solve_async(1, y, x)
        want, bad = oracle.factor_serial(rs, col, v.copy(), diag, 0.0, False)
        assert bad < 0 and dv.read_row_slot(d.err) == -1
        assert np.array_equal(d.host_val(), want)
        yo = oracle.solve_forward(rs, col, want, b)
        xo, _ = oracle.solve_backward(rs, col, want, diag, yo)
        assert np.array_equal(dv.host_f64(y, n), yo)
        assert np.array_equal(dv.host_f64(x, n), xo)
    if mode == "on":
        assert all(d.region_stream(s) is not None for s in ("factor", "fwd", "bwd"))
    dv.check_hang()


@pytest.mark.parametrize("m", [1, 7, 8, 9, 31, 4096 + 5, 1 << 20])
def test_pack_values_gather(m):
    """jv_pack_values: dst[e] = src[sidx[e]], 0 where sidx < 0, every length
    (full tiles and a partial one)."""
    from paper_1812_06160_b200 import _lib
    from paper_1812_06160_b200.device import ptr, stream

    t = dv.torch()
    rng = np.random.default_rng(m)
    src = rng.standard_normal(3 * m + 1)
    sidx = rng.integers(-1, src.size, m).astype(np.int32)
    want = np.where(sidx >= 0, src[np.maximum(sidx, 0)], 0.0)
    s_d = dv.f64(src)
    i_d = t.from_numpy(sidx).cuda()
    out = t.full((m + 2,), 7.0, dtype=t.float64, device="cuda")
    _lib.call("jv_pack_values", m, ptr(i_d), ptr(s_d), ptr(out), stream())
    got = out.cpu().numpy()
    assert np.array_equal(got[:m], want)
    assert np.all(got[m:] == 7.0)   # nothing written past m


@pytest.mark.parametrize("m1,m2", [(0, 0), (0, 9), (13, 0), (5000, 3), (1 << 21, 1 << 20),
                                   (7, 1 << 22)])
def test_pack_values2_two_jobs_and_reset(m1, m2):
    """jv_pack_values2: both gathers (the launch grid split between them,
    capped) and the error-row reset in one launch."""
    from paper_1812_06160_b200 import _lib
    from paper_1812_06160_b200.device import ptr, stream

    t = dv.torch()
    rng = np.random.default_rng(m1 * 7 + m2)
    jobs = []
    for m in (m1, m2):
        src = rng.standard_normal(2 * m + 3)
        sidx = rng.integers(-1, src.size, m).astype(np.int32)
        want = np.where(sidx >= 0, src[np.maximum(sidx, 0)], 0.0)
        out = t.full((m + 1,), 5.0, dtype=t.float64, device="cuda")
        jobs.append((dv.f64(src), t.from_numpy(sidx).cuda(), out, want, m))
    slot = t.zeros(1, dtype=t.int32, device="cuda")
    (s1, i1, o1, _, _), (s2, i2, o2, _, _) = jobs
    _lib.call("jv_pack_values2", m1, ptr(i1), ptr(s1), ptr(o1), m2, ptr(i2), ptr(s2), ptr(o2),
              ptr(slot), stream())
    for _, _, out, want, m in jobs:
        got = out.cpu().numpy()
        assert np.array_equal(got[:m], want) and got[m] == 5.0
    assert dv.read_row_slot(slot) == -1   # reset to "no row"
