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
