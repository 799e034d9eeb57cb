"""CPU: the oracle restatement is pinned to the reference's own outputs
(golden vectors from tests/golden/make_golden.py)."""

import math

import numpy as np
import pytest

from conftest import unb64, unhex
from oracle import np_oracle as orc
from paper_2404_08867_b200 import parse
from paper_2404_08867_b200.configs import make_config


def test_points_match_reference_bitwise(golden):
    for case in golden["points"]:
        n = int(case["n"])
        z = [int(c) for c in case["z"]]
        got = orc.points_block(n, z, case["start"], case["stop"])
        want = unb64(case["data"], case["shape"])
        assert np.array_equal(got.view(np.uint64), want.view(np.uint64)), case["tag"]


def test_points_overflow_guard():
    with pytest.raises(OverflowError):
        orc.points_block(2**54, [1], 0, 1)


@pytest.mark.parametrize("tag", ["const_2p5", "dual_mode", "nondual_mode", "expxy_101", "expxy_40001",
                                 "sinsq_2027", "gaussian5", "ratprod4", "invpow3", "expsq4", "coslin6",
                                 "expalt7", "poly_mix", "recip_sum", "sin_of_prod", "cfg1", "cfg2"])
def test_slr_matches_reference(golden, tag):
    case = next(c for c in golden["slr"] if c["tag"] == tag)
    n = int(case["n"])
    got = orc.slr_value(case["text"], n, [int(c) for c in case["z"]])
    want = unhex(case["value"])
    assert abs(got - want) <= 1e-13 * max(abs(want), 1e-3), (tag, got, want)


def test_cfg5_range_restatement(golden):
    case = next(c for c in golden["slr"] if c["tag"] == "cfg5_range_0_16384")
    got = orc.slr_sum(case["text"], int(case["n"]), [int(c) for c in case["z"]], 0, 1 << 14)
    assert abs(got - unhex(case["range_sum"])) <= 1e-12 * unhex(case["range_sum"])


def test_axis_counts_and_normalize_match_reference(golden):
    for case in golden["mdi"]:
        if "counts" not in case:
            continue
        n, a, d = int(case["n"]), case["a"], case["d"]
        z = [a**j for j in range(d)]
        counts = orc.axis_counts(n, z)
        assert [str(c) for c in counts] == case["counts"], case["tag"]
        raw = unhex(case["raw"])
        assert orc.normalize(raw, counts) == unhex(case["value"]), case["tag"]


def test_direct_tensor_sum_matches_reference(golden):
    checked = 0
    for case in golden["mdi"]:
        if "direct_sum" not in case:
            continue
        counts = [int(c) for c in case["counts"]]
        if math.prod(counts) > 200_000:
            continue
        got = orc.direct_tensor_sum(case["text"], orc.midpoint_nodes(counts))
        want = unhex(case["direct_sum"])
        assert abs(got - want) <= 1e-13 * abs(want), case["tag"]
        checked += 1
    assert checked > 100


def test_separable_closed_form_matches_reference_mdi(golden):
    # separable MDI-LR == product of per-direction cluster sums
    case = next(c for c in golden["mdi"] if c["tag"] == "cfg4")
    cfg = make_config(4)
    c = np.asarray(cfg.c)
    w = np.asarray(cfg.w)
    fns = [(lambda y, cj=cj, wj=wj: 1.0 / (cj ** -2 + (y - wj) ** 2)) for cj, wj in zip(c, w)]
    log_raw, sign = orc.separable_log_sum(fns, [cfg.mdi_a] * cfg.d)
    assert sign == 1.0
    assert abs(log_raw - unhex(case["log_raw"])) <= 1e-12 * abs(log_raw)


def test_configs_are_seeded_as_documented(golden):
    # the seeded a of the plain-sum lattices and the integrand texts the golden vectors used
    for cid in (1, 2, 3):
        cfg = make_config(cid)
        case = next(c for c in golden["slr"] if c["tag"] == f"cfg{cid}")
        assert case["text"] == cfg.text
        assert int(case["z"][1]) == cfg.plain_a
    assert make_config(3).plain_a == 811507


def test_mc_oracle_pinned_to_reference():
    # quad.mc_integrate values and the first rows of each stream, frozen from the reference
    import numpy as np
    import paper_2404_08867_b200 as lq
    from conftest import load_golden, unb64, unhex
    from oracle import np_oracle
    for case in load_golden("mc"):
        got = np_oracle.mc_value(case["text"], case["d"], case["n"], case["seed"])
        assert abs(got - unhex(case["value"])) <= 1e-13 * abs(unhex(case["value"])), case["tag"]
        first = unb64(case["first_rows"], case["first_shape"])
        st = np.random.default_rng(case["seed"]).bit_generator.state["state"]
        d = case["d"]
        for i in (0, 1, first.shape[0] - 1):
            for j in range(d):
                assert np_oracle.pcg64_draw(st["state"], st["inc"], i * d + j) == first[i, j], (case["tag"], i, j)


def test_oracle_eval_matches_reference_eval_on_parser_corpus():
    """The oracle's own literal evaluator (np_oracle.eval_array -> np_expr, no
    product code) against the reference's exprcore.eval frozen at three points
    per accepted text of the parser corpus (tests/golden/parser.json).  The
    reference canonicalises before evaluating (angle addition, quadratic
    expansion, constant folding), the oracle evaluates the text as written:
    1e-10, or 1e-8 for constant texts whose huge trig arguments amplify the
    folding order."""
    import math
    from oracle import np_oracle
    from conftest import load_golden, unhex
    n = 0
    for case in load_golden("parser"):
        if "error" in case:
            continue
        d = case["d"]
        tol = 1e-10 if "x[" in case["text"] else 1e-8
        for pt, want in zip(case["points"], case["values"]):
            if not want.startswith(("0x", "-0x", "inf", "-inf", "nan")):
                continue   # the reference raised at this point (e.g. a zero base to a negative power)
            assign = {j + 1: np.array([unhex(v)]) for j, v in enumerate(pt)}
            with np.errstate(all="ignore"):
                got = float(np.asarray(np_oracle.eval_array(case["text"], d, assign)).reshape(-1)[0])
            w = unhex(want)
            assert got == w or math.isclose(got, w, rel_tol=tol, abs_tol=1e-300) or (math.isnan(got) and math.isnan(w)), \
                (case["text"], got, w)
            n += 1
    assert n > 800


def test_oracle_takes_text_only():
    """The oracle shares nothing with the product front end: a product Expr is
    refused, and nothing under oracle/ imports the product package."""
    import os
    import re
    import paper_2404_08867_b200 as lq
    from oracle import np_oracle
    with pytest.raises(TypeError):
        np_oracle.eval_array(lq.parse("x[1]", 1), 1, {1: np.array([0.5])})
    here = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "oracle")
    for name in os.listdir(here):
        if name.endswith(".py"):
            src = open(os.path.join(here, name)).read()
            assert not re.search(r"^\s*(from|import)\s+paper_2404_08867_b200", src, re.M), name
