"""Benchmark-suite rows (suites.run_row, the caller side of the path) on the
GPU against the reference's own rows (tests/golden/suites.json and
suites7.json, frozen from latquad.bench): same skip decisions, values within
1e-10 (Monte-Carlo rows: same PCG64 stream, so summation-order rounding
only).  Suite test7 is checked on its d <= 10 rows (invpow's levels collapse
through lq_mdi_linform; the reference needs ~7 min for d = 10 alone)."""

import math
import os

import pytest

from conftest import GOLDEN, load_golden, unhex

pytestmark = pytest.mark.gpu


def _check(rec, want, tag):
    assert rec.status == want["status"], tag
    if want["value"] is None:
        assert rec.value is None, tag
        return
    v = unhex(want["value"])
    assert math.isclose(rec.value, v, rel_tol=1e-10, abs_tol=1e-300), (tag, rec.value, v)
    if want["reference"] is not None:
        assert rec.reference == unhex(want["reference"]), tag


@pytest.mark.parametrize("suite", ["test1", "test2", "test3", "test5"])
def test_suite_rows_match_reference(suite, tmp_path):
    from paper_2404_08867_b200 import suites
    rows = [r for r in load_golden("suites") if r["suite"] == suite]
    recs = suites.run_suite(suite, tmp_path / f"{suite}.csv")
    assert len(recs) == len(rows)
    for rec, want in zip(recs, rows):
        _check(rec, want, (suite, rec.method, rec.integrand, rec.d, rec.n, rec.a))
    from paper_2404_08867_b200.fits import read_rows
    assert len(read_rows(tmp_path / f"{suite}.csv")) >= 1


@pytest.mark.skipif(not os.path.exists(os.path.join(GOLDEN, "suites7.json")), reason="suites7.json not frozen")
def test_suite7_rows_up_to_d10_match_reference():
    from paper_2404_08867_b200 import suites
    rows = load_golden("suites7")
    assert {r["integrand"] for r in rows} >= {"invpow", "expalt", "ratprod", "gaussian", "coslin", "expsq"}
    for want in rows:
        spec = (want["method"], want["integrand"], want["d"], int(want["n"]), want["a"])
        assert spec in suites.suite_specs("test7")
        _check(suites.run_row(spec), want, spec)
