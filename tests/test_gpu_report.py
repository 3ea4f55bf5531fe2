"""The schema-compatible device report (report.run_report): valid against
the reference's report schema (restated), serial digest equal to the
reference's own factor values, determinism across independent runs."""

import hashlib
import json

import numpy as np
import pytest

import report_schema_check as R

pytestmark = pytest.mark.gpu

jv = pytest.importorskip("paper_1812_06160_b200")
from paper_1812_06160_b200.report import run_report  # noqa: E402


def test_report_digest_is_the_reference_factor(golden):
    g = golden.case("poisson3d_5")
    n = g["a_rs"].size - 1
    a = jv.CsrMatrix(n, g["a_rs"], g["a_col"], g["a_val"])
    r = run_report(a, "poisson3d_5", threads=[1, 2, 4], repeats=2)
    R.check_report(json.loads(json.dumps(r)))
    want = hashlib.sha256(np.ascontiguousarray(g["fval"]).tobytes()).hexdigest()
    assert r["digests"]["serial"] == want
    assert r["determinism_ok"]
    assert r["partition"]["n_upper"] == int(g["n_upper"])
    assert r["levels"]["num_levels"] == int(g["level_of"].max()) + 1


@pytest.mark.parametrize("solver", ["pcg", "gmres"])
def test_report_with_tail_and_krylov(solver):
    a = jv.poisson2d(24) if solver == "pcg" else jv.convdiff2d(20, seed=2)
    r = run_report(a, "m", order="rcm", min_level_rows=40, threads=[1, 8], solver=solver,
                   tol=1e-8, repeats=2)
    R.check_report(json.loads(json.dumps(r)))
    assert r["partition"]["rows_excluded"] > 0 and r["partition"]["method"] == "er"
    assert r["timings"]["factor_lower"]["1"] is not None
    assert r["determinism_ok"]
    assert r["krylov"]["converged"]
