"""Pin the Krylov oracle (oracle.pcg / oracle.gmres) against the reference's
own krylov.py runs (tests/golden/krylov.npz, made by
tests/golden/make_krylov_golden.py), including acceptance criterion 7
(Poisson 64x64, tol 1e-6: ILU(0)-PCG 43 < CG 104; pkg/test_output.txt:23).
CPU only; the device solvers are checked against the same fixtures in
tests/test_gpu_krylov.py."""

import json
import os

import numpy as np
import pytest

import oracle
from conftest import GOLDEN

Z = np.load(os.path.join(GOLDEN, "krylov.npz"))
NAMES = [str(s) for s in Z["_names"]]


def case(name):
    pre = name + "/"
    g = {k[len(pre):]: Z[k] for k in Z.files if k.startswith(pre)}
    g["meta"] = json.loads(str(g["meta"][0]))
    return g


def oracle_ilu(rs, col, val, k):
    """Identity-ordered ILU(k) factors through the oracle (symbolic.py +
    factor_serial restated)."""
    n = rs.size - 1
    if k == 0:
        frs, fcol = rs, col
    else:
        frs, fcol, _ = oracle.iluk_pattern(rs, col, k)
    fv, diag, covered, miss = oracle.assemble(n, rs, col, val, frs, fcol)
    assert covered and miss < 0
    fval, bad = oracle.factor_serial(frs, fcol, fv, diag)
    assert bad < 0
    return lambda r: oracle.ilu_apply(frs, fcol, fval, diag, r)


@pytest.mark.parametrize("name", NAMES)
def test_oracle_krylov_matches_reference(name):
    g = case(name)
    m = g["meta"]
    pre = None if m["k"] is None else oracle_ilu(g["a_rs"], g["a_col"], g["a_val"], m["k"])
    if m["method"] == "pcg":
        x, it, ok, hist = oracle.pcg(g["a_rs"], g["a_col"], g["a_val"], g["b"], pre,
                                     tol=m["tol"], maxit=m["maxit"])
    else:
        x, it, ok, hist = oracle.gmres(g["a_rs"], g["a_col"], g["a_val"], g["b"], pre,
                                       restart=m["restart"], tol=m["tol"], maxit=m["maxit"])
    assert it == int(g["iterations"]) and ok == bool(g["converged"])
    assert np.allclose(hist, g["history"], rtol=1e-9, atol=1e-15)
    assert np.allclose(x, g["x"], rtol=1e-9, atol=1e-12)


def test_criterion_7_known_answer():
    """The reference's published numbers: CG 104, ILU(0)-PCG 43."""
    assert int(case("c7_cg")["iterations"]) == 104
    assert int(case("c7_ilu0_pcg")["iterations"]) == 43
