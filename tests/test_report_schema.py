"""CPU: the restated report schema (tests/report_schema_check.py) matches
the reference's own schema file (pkg/docs/report_schema.json) when the
reference is present (build container only)."""

import json
import os

import pytest

import report_schema_check as R

SCHEMA = "/root/reference/pkg/docs/report_schema.json"


@pytest.mark.skipif(not os.path.exists(SCHEMA), reason="reference schema not present")
def test_restated_schema_matches_reference():
    s = json.load(open(SCHEMA))
    p = s["properties"]
    assert s["required"] == R.TOP
    assert p["config"]["required"] == R.CONFIG
    assert p["matrix"]["required"] == R.MATRIX
    assert p["levels"]["required"] == R.LEVELS
    assert p["partition"]["required"] == R.PARTITION
    assert p["krylov"]["oneOf"][1]["required"] == R.KRYLOV
    assert p["digests"]["required"] == R.DIGESTS
    assert p["schema_version"]["const"] == 1


def test_checker_rejects_missing_keys():
    with pytest.raises(AssertionError):
        R.check_report({"schema_version": 1})
