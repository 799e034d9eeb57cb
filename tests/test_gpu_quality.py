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


def _terms(lq, n, z, gamma, beta, alpha=2):
    """The per-point products exactly as the kernel forms them: numpy's
    points_block / bernoulli_poly / 1 + g (B + beta), multiplied left to right."""
    import numpy as np
    from oracle import np_oracle as orc
    x = orc.points_block(n, list(z), 0, n)
    out = np.ones(n)
    for j in range(len(z)):
        out = out * (1.0 + gamma[j] * (lq.bernoulli_poly(x[:, j], alpha) + beta))
    return out


def test_quality_sums_are_exact_and_order_free(lq):
    """The Bernoulli-product sums are exact fixed-point sums rounded once
    (Fix3): equal to math.fsum of the same terms, and bit-identical for
    rules whose terms are permutations of each other -- reflections c <-> n-c,
    and coordinate swaps under equal weights -- the exact ties the
    reference gets by sorting its terms (lattice.py:236-239, 284)."""
    import math
    for n, c in [(9, 2), (17, 5), (101, 37), (1009, 400), (65537, 12345)]:
        w = lq.WeightModel.default(2)
        a = lq.shift_avg_wce_sq(lq.LatticeRule(n, (1, c)), w)
        b = lq.shift_avg_wce_sq(lq.LatticeRule(n, (1, n - c)), w)
        assert a == b, (n, c, a, b)
        t = _terms(lq, n, (1, c), w.gamma, w.beta)
        anchor = float(__import__("numpy").prod(1.0 + __import__("numpy").asarray(w.gamma) * w.beta))
        assert a == math.fsum(t) / n - anchor, (n, c)
        eq = lq.WeightModel.unanchored((0.7, 0.7, 0.7))
        s1 = lq.shift_avg_wce_sq(lq.LatticeRule(n, (1, c, (c * c) % n)), eq)
        s2 = lq.shift_avg_wce_sq(lq.LatticeRule(n, ((c * c) % n, 1, c)), eq)
        assert s1 == s2, (n, c)
        p1 = lq.p_alpha(lq.LatticeRule(n, (1, c)), 4)
        p2 = lq.p_alpha(lq.LatticeRule(n, (1, n - c)), 4)
        assert p1 == p2


def test_cbc_matches_exhaustive_per_step_search(lq):
    """Exhaustive per-step CBC over shift_avg_wce_sq with strict < (smallest
    candidate keeps exact ties) gives the same vectors as cbc_construct --
    the reference's own check (tests/test_lattice.py TestCbcConstruct), here
    with this package's measure on both sides."""
    import math
    for n in (5, 8, 9, 12, 13, 16, 17, 31, 64):
        for d in (2, 3, 4):
            w = lq.WeightModel.default(d)
            cands = [c for c in range(1, n) if math.gcd(c, n) == 1]
            z = [1]
            for k in range(2, d + 1):
                best, best_val = None, None
                for c in cands:
                    val = lq.shift_avg_wce_sq(lq.LatticeRule(n, tuple(z) + (c,)), w.prefix(k))
                    if best_val is None or val < best_val:
                        best, best_val = c, val
                z.append(best)
            assert lq.cbc_construct(n, d, w).z == tuple(z), (n, d)
