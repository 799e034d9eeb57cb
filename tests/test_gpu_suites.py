"""Benchmark-suite rows (suites.run_row, the caller side of the path) on the
GPU against the reference's own rows (tests/golden/suites.json, frozen from
latquad.bench): same skip decisions, values within 1e-10 (Monte-Carlo rows:
same PCG64 stream, so summation-order rounding only)."""

import math

import pytest

from conftest import load_golden, unhex

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("suite", ["test1", "test2", "test3", "test5"])
def test_suite_rows_match_reference(suite, tmp_path):
    from paper_2404_08867_b200 import suites
    rows = [r for r in load_golden("suites") if r["suite"] == suite]
    recs = suites.run_suite(suite, tmp_path / f"{suite}.csv")
    assert len(recs) == len(rows)
    for rec, want in zip(recs, rows):
        tag = (suite, rec.method, rec.integrand, rec.d, rec.n, rec.a)
        assert rec.status == want["status"], tag
        if want["value"] is None:
            assert rec.value is None, tag
            continue
        v = unhex(want["value"])
        assert math.isclose(rec.value, v, rel_tol=1e-10, abs_tol=1e-300), (tag, rec.value, v)
        if want["reference"] is not None:
            assert rec.reference == unhex(want["reference"]), tag
    from paper_2404_08867_b200.fits import read_rows
    assert len(read_rows(tmp_path / f"{suite}.csv")) >= 1
