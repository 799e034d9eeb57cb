"""GPU: lattice quality measures and constructions against the reference's
own outputs (tests/golden/quality.json; lattice.py:140-311)."""

import warnings

import pytest

from conftest import unhex

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lq():
    import paper_2404_08867_b200 as m
    return m


def _rule(lq, c):
    return lq.LatticeRule(int(c["n"]), tuple(int(v) for v in c["z"]))


def test_p_alpha_matches_reference(lq, golden_quality):
    for c in golden_quality:
        if c["tag"] not in ("p_alpha2", "p_alpha4"):
            continue
        with warnings.catch_warnings(record=True) as w:
            warnings.simplefilter("always")
            got = lq.p_alpha(_rule(lq, c), c["alpha"])
        want = unhex(c["value"])
        assert abs(got - want) <= 1e-10 * max(abs(want), 1e-6), (c, got, want)
        assert bool(w) == c["warned"]


def test_shift_avg_wce_matches_reference(lq, golden_quality):
    for c in golden_quality:
        if c["tag"] != "wce":
            continue
        wm = None
        if c["gamma"] is not None:
            wm = lq.WeightModel(tuple(unhex(g) for g in c["gamma"]), unhex(c["beta"]))
        got = lq.shift_avg_wce_sq(_rule(lq, c), wm)
        want = unhex(c["value"])
        assert abs(got - want) <= 1e-10 * abs(want) + 1e-15, (c["n"], got, want)


def test_cbc_matches_reference(lq, golden_quality):
    for c in golden_quality:
        if c["tag"] == "cbc":
            assert lq.cbc_construct(c["n"], c["d"]).z == tuple(c["z"]), c
        elif c["tag"] == "cbc_anchored":
            wm = lq.WeightModel(tuple(unhex(g) for g in c["gamma"]), unhex(c["beta"]))
            assert lq.cbc_construct(c["n"], c["d"], wm).z == tuple(c["z"]), c


def test_korobov_search_matches_reference(lq, golden_quality):
    for c in golden_quality:
        if c["tag"] == "korobov_search":
            r = lq.korobov_search(c["n"], c["d"], criterion=c["criterion"])
            assert r.z[1] == c["a"], (c, r.z[:2])


def test_validation_mirrors_reference(lq):
    with pytest.raises(ValueError):
        lq.p_alpha(lq.LatticeRule(5, (1,)), 3)
    with pytest.raises(ValueError):
        lq.cbc_construct(1, 3)
    with pytest.raises(ValueError):
        lq.korobov_search(101, 3, criterion="nope")
    with pytest.raises(ValueError):
        lq.shift_avg_wce_sq(lq.LatticeRule(8, (1, 3)), lq.WeightModel((1.0,)))
