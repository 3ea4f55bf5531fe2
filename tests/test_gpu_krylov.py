"""Device Krylov driver (krylov.py): PCG / GMRES over the GPU spmv and the
resident ILU preconditioner, against the numpy restatement of the
reference's krylov.py in oracle/ (iteration counts, solutions) and the
reference's own behavioural cases (exact preconditioners, zero RHS,
breakdown, Krylov optimality, ordering experiment)."""

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

jv = pytest.importorskip("paper_1812_06160_b200")


def ilu(a, k=0):
    pat, _ = jv.iluk_pattern(a.pattern, k)
    f = jv.assemble_factors(a, pat, jv.Permutation.identity(a.n))
    jv.factor_serial(f)
    return f


def oracle_precond(f):
    rs, col, val, dg = f.pattern.row_start, f.pattern.col, f.val, f.diag_pos
    return lambda r: oracle.ilu_apply(rs, col, val, dg, r)


def test_pcg_identity_and_zero_rhs():
    a = jv.CsrMatrix.from_dense(np.eye(6))
    res = jv.pcg(a, np.arange(2.0, 8.0))
    assert res.converged and res.iterations == 1 and np.allclose(res.x, np.arange(2.0, 8.0))
    res = jv.pcg(jv.tridiag(7), np.zeros(7))
    assert res.converged and res.iterations == 0 and np.array_equal(res.x, np.zeros(7))


def test_pcg_exact_ilu_one_iteration():
    a = jv.tridiag(50)
    res = jv.pcg(a, np.linspace(-1.0, 2.0, 50), jv.ilu_preconditioner(ilu(a)), tol=1e-10)
    assert res.converged and res.iterations == 1


@pytest.mark.parametrize("kind", ["none", "device", "host"])
def test_pcg_matches_oracle(kind):
    a = jv.poisson2d(24)
    b = jv.spmv(a, np.linspace(0.5, 1.5, a.n))
    f = ilu(a)
    pre = {"none": None, "device": jv.ilu_preconditioner(f),
           "host": (lambda r: jv.apply_preconditioner(f, r))}[kind]
    res = jv.pcg(a, b, pre, tol=1e-9, maxit=500)
    x, it, ok, hist = oracle.pcg(a.row_start, a.col, a.val, b,
                                 None if kind == "none" else oracle_precond(f), tol=1e-9, maxit=500)
    assert res.converged and ok
    assert res.iterations == it
    assert len(res.residual_history) == res.iterations + 1
    assert np.allclose(res.residual_history, hist, rtol=1e-6, atol=1e-14)
    assert np.allclose(res.x, x, rtol=1e-8, atol=1e-10)
    true_rel = np.linalg.norm(b - jv.spmv(a, res.x)) / np.linalg.norm(b)
    assert abs(true_rel - res.residual_history[-1]) <= 1e-9


def test_ilu_preconditioning_cuts_pcg_iterations():
    a = jv.poisson2d(40)
    b = jv.spmv(a, np.ones(a.n))
    plain = jv.pcg(a, b, tol=1e-8, maxit=1000)
    pre = jv.pcg(a, b, jv.ilu_preconditioner(ilu(a)), tol=1e-8, maxit=1000)
    assert plain.converged and pre.converged
    assert pre.iterations < 0.6 * plain.iterations


def test_pcg_breakdown_reported():
    a = jv.CsrMatrix.from_dense([[2.0, 0.0], [0.0, -3.0]])
    with pytest.raises(jv.BreakdownError) as exc:
        jv.pcg(a, np.array([1.0, 1.0]))
    assert exc.value.iteration == 1


def test_gmres_identity_and_exact_preconditioner():
    a = jv.CsrMatrix.from_dense(np.eye(5))
    res = jv.gmres(a, np.array([1.0, -2.0, 3.0, 0.5, 4.0]))
    assert res.converged and res.iterations == 1
    d = jv.CsrMatrix.from_dense(np.diag(np.arange(1.0, 21.0)))
    res = jv.gmres(d, np.ones(20), jv.ilu_preconditioner(ilu(d)), tol=1e-10)
    assert res.converged and res.iterations == 1


@pytest.mark.parametrize("restart", [50, 7])
def test_gmres_matches_oracle(restart):
    a = jv.convdiff2d(16, seed=3)
    b = jv.spmv(a, np.ones(a.n))
    f = ilu(a)
    res = jv.gmres(a, b, jv.ilu_preconditioner(f), restart=restart, tol=1e-9, maxit=400)
    x, it, ok, hist = oracle.gmres(a.row_start, a.col, a.val, b, oracle_precond(f),
                                   restart=restart, tol=1e-9, maxit=400)
    assert res.converged == ok and res.iterations == it
    assert np.allclose(res.residual_history, hist, rtol=1e-6, atol=1e-14)
    assert np.allclose(res.x, x, rtol=1e-7, atol=1e-10)


def test_gmres_residuals_krylov_optimal():
    """Unpreconditioned GMRES residuals equal the least-squares optimum over
    K_m(A, b) (the reference's Krylov-optimality property)."""
    a = jv.convdiff2d(6, seed=1)
    b = np.linspace(1.0, 2.0, a.n)
    res = jv.gmres(a, b, restart=a.n, tol=1e-14, maxit=12)
    dense = a.to_dense()
    bn = np.linalg.norm(b)
    for m in range(1, 8):
        cols = [b]
        for _ in range(m - 1):
            cols.append(dense @ cols[-1])
        V = np.stack(cols, axis=1)
        y, *_ = np.linalg.lstsq(dense @ V, b, rcond=None)
        opt = np.linalg.norm(b - dense @ (V @ y)) / bn
        assert abs(res.residual_history[m] - opt) <= 1e-8


def test_iteration_experiment_orderings():
    a = jv.poisson2d(20)
    rows = jv.iteration_experiment(a, orderings=[
        ("natural", None, False),
        ("natural+LS", None, True),
        ("rcm", jv.rcm_order(a.pattern), False),
    ], tol=1e-8)
    assert [r["method"] for r in rows] == ["pcg"] * 3
    assert all(r["converged"] for r in rows)
    counts = [r["iterations"] for r in rows]
    assert all(c is not None and 5 < c < 200 for c in counts)
    un = jv.convdiff2d(10, seed=2)
    rows = jv.iteration_experiment(un, orderings=[("natural", None, False)])
    assert rows[0]["method"] == "gmres" and rows[0]["converged"]
