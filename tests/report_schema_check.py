"""Restatement of the reference report schema (pkg/docs/report_schema.json,
version 1) as plain checks, used by the report tests (no jsonschema
dependency; tests/test_report_schema.py pins the restated key lists against
the reference's schema file when it is present)."""

import re

TOP = ["schema_version", "config", "matrix", "levels", "partition", "timings", "speedups",
       "solve_speedups_vs_csrls", "krylov", "digests", "determinism_ok"]
CONFIG = ["matrix", "order", "levels_on", "k", "tau", "milu", "lower", "min_level_rows",
          "density_factor", "tile_size", "threads", "solver", "restart", "tol", "maxit", "repeats"]
MATRIX = ["name", "n", "nnz", "mean_row_nnz"]
LEVELS = ["num_levels", "min_rows", "max_rows", "median_rows"]
PARTITION = ["cut_level", "num_upper_levels", "n_upper", "rows_excluded", "method"]
KRYLOV = ["method", "iterations", "converged", "final_relative_residual", "stopping_rule"]
DIGESTS = ["serial", "factor", "solve"]
SHA = re.compile(r"^[0-9a-f]{64}$")
WKEY = re.compile(r"^[0-9]+$")


def check_report(r):
    assert set(r) == set(TOP), set(r) ^ set(TOP)
    assert r["schema_version"] == 1
    assert set(CONFIG) <= set(r["config"])
    c = r["config"]
    assert c["order"] in ("natural", "rcm", "file") and c["levels_on"] in ("A", "AplusAT")
    assert c["lower"] in ("auto", "sr", "er", "none") and c["solver"] in ("none", "pcg", "gmres")
    assert all(isinstance(t, int) and t >= 1 for t in c["threads"])
    assert set(MATRIX) <= set(r["matrix"]) and set(LEVELS) <= set(r["levels"])
    assert set(PARTITION) <= set(r["partition"])
    assert r["partition"]["method"] in ("sr", "er", "none")
    for sec in ("timings", "speedups", "solve_speedups_vs_csrls"):
        for row in r[sec].values():
            for k, v in row.items():
                assert WKEY.match(str(k)) and (v is None or isinstance(v, (int, float)))
    if r["krylov"] is not None:
        assert set(KRYLOV) <= set(r["krylov"])
        assert r["krylov"]["stopping_rule"] == "relative_residual"
    d = r["digests"]
    assert set(DIGESTS) <= set(d) and SHA.match(d["serial"])
    assert all(WKEY.match(str(k)) and SHA.match(v) for k, v in d["factor"].items())
    for row in d["solve"].values():
        assert all(WKEY.match(str(k)) and SHA.match(v) for k, v in row.items())
    assert isinstance(r["determinism_ok"], bool)
