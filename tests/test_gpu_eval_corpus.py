"""GPU: every accepted text of the reference-frozen parser corpus
(tests/golden/parser.json: fixed quirk cases, 400 fuzzed texts, the integrand
corpus) parsed by the product and evaluated by the GPU bytecode interpreter
(k_prog_tensor through lq_tensor_sum on a one-node grid at the frozen point)
against the reference's exprcore.eval at that point (the
product front end meets reference values without going through the oracle)."""

import math

import pytest

from conftest import load_golden, unhex

pytestmark = pytest.mark.gpu

CASES = [c for c in load_golden("parser") if "error" not in c]


def test_gpu_bytecode_matches_reference_eval():
    import paper_2404_08867_b200 as lq
    from paper_2404_08867_b200.transform import AxisGridSet
    checked = 0
    for case in CASES:
        text, d = case["text"], case["d"]
        f = lq.parse(text, d)
        if not lq.free_vars(f):
            continue
        for pt, want in zip(case["points"], case["values"]):
            x = [unhex(v) for v in pt]
            grid = AxisGridSet(tuple((v,) for v in x), (1,) * d, None, None)
            got = lq.direct_tensor_sum(f, grid)
            w = unhex(want)
            assert got == w or math.isclose(got, w, rel_tol=1e-10, abs_tol=1e-300), (text, x, got, w)
            checked += 1
    assert checked > 300, checked      # texts with coordinates, three points each


def test_gpu_eval_array_matches_reference_eval():
    """eval_array (k_prog_eval through lq_eval_array): the corpus texts over
    all three frozen points at once (one column per coordinate, m = 3) against
    the reference's values, 1e-10 (reference-raised points are skipped)."""
    import numpy as np
    import paper_2404_08867_b200 as lq
    checked = 0
    for case in CASES:
        text, d = case["text"], case["d"]
        f = lq.parse(text, d)
        if not lq.free_vars(f):
            assert lq.eval_array(f, {}) == lq.eval(f, {})
            continue
        keep = [i for i, w in enumerate(case["values"]) if w.startswith(("0x", "-0x", "inf", "-inf", "nan"))]
        if not keep:
            continue
        pts = np.array([[unhex(v) for v in case["points"][i]] for i in keep])
        with np.errstate(all="ignore"):
            got = lq.eval_array(f, {j + 1: pts[:, j] for j in range(d)})
        assert got.shape == (len(keep),)
        for g, i in zip(got, keep):
            w = unhex(case["values"][i])
            assert g == w or math.isclose(g, w, rel_tol=1e-10, abs_tol=1e-300) or (math.isnan(g) and math.isnan(w)), \
                (text, g, w)
            checked += 1
    assert checked > 300, checked      # texts with coordinates, three points each


def test_gpu_eval_array_shapes_and_errors():
    """Broadcasting (column against scalar, 2-D blocks), empty input, a
    missing coordinate, and 2^20 rows of config 3's integrand against the
    oracle's literal evaluator (1e-13)."""
    import numpy as np
    import paper_2404_08867_b200 as lq
    from oracle import np_oracle as orc
    from paper_2404_08867_b200.configs import make_config
    f = lq.parse("exp(x[1]) * cos(x[2] + 2*x[3])", 3)
    a = np.linspace(0.0, 1.0, 7)
    got = lq.eval_array(f, {1: a, 2: 0.25, 3: a[::-1]})
    want = np.exp(a) * np.cos(0.25 + 2 * a[::-1])
    assert got.shape == (7,) and np.allclose(got, want, rtol=1e-14, atol=0)
    blk = np.random.default_rng(3).random((5, 4, 3))
    got2 = lq.eval_array(f, {j + 1: blk[..., j] for j in range(3)})
    assert got2.shape == (5, 4) and np.allclose(got2, np.exp(blk[..., 0]) * np.cos(blk[..., 1] + 2 * blk[..., 2]),
                                                rtol=1e-14, atol=0)
    assert isinstance(lq.eval_array(f, {1: 0.1, 2: 0.2, 3: 0.3}), float)
    assert lq.eval_array(f, {1: np.zeros(0), 2: np.zeros(0), 3: np.zeros(0)}).shape == (0,)
    with pytest.raises(lq.UnassignedVariableError):
        lq.eval_array(f, {1: a, 3: a})
    cfg = make_config(3)
    g = lq.parse(cfg.text, cfg.d)
    pts = orc.points_block(cfg.plain_n, [cfg.plain_a ** j for j in range(cfg.d)], 0, 1 << 20)
    cols = {j + 1: pts[:, j] for j in range(cfg.d)}
    got3 = lq.eval_array(g, cols)
    want3 = orc.eval_array(cfg.text, cfg.d, cols)
    assert np.allclose(got3, want3, rtol=1e-13, atol=0)
