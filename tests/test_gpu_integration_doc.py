"""GPU: the reference-side binding INTEGRATION.md shows a latquad maintainer
(its `latquad/_gpu.py` ctypes snippet and `level_collapse_mean`) runs as
written against liblq.so and gives the package's own results: bit-identical
points, the OverflowError mapping, and the level-collapse grid mean."""

import os
import re

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def snippet():
    from paper_2404_08867_b200 import _native as N
    N.lib()
    text = open(os.path.join(REPO, "INTEGRATION.md")).read()
    blocks = re.findall(r"```python\n(.*?)```", text, flags=re.S)
    gpu = next(b for b in blocks if b.startswith("# latquad/_gpu.py"))
    lcm = next(b for b in blocks if b.startswith("def level_collapse_mean"))
    ns = {}
    exec(compile(gpu.replace('"liblq.so"', repr(N.LIB_PATH)), "INTEGRATION.md:_gpu.py", "exec"), ns)
    exec(compile(lcm, "INTEGRATION.md:level_collapse_mean", "exec"), ns)
    return ns


def test_points_block_binding(snippet):
    import paper_2404_08867_b200 as lq
    for n, a, d in ((1009, 17, 8), (65521, 4321, 30), (2147483647, 1440510675, 12)):
        rule = lq.korobov_vector(a, n, d)
        got = snippet["points_block"](rule, 5, 700)
        assert np.array_equal(got, lq.points_block(rule, 5, 700))
    big = lq.LatticeRule(2**54 + 1, (1, 3))
    with pytest.raises(OverflowError):
        snippet["points_block"](big, 0, 4)


def test_level_collapse_binding(snippet):
    import paper_2404_08867_b200 as lq
    from paper_2404_08867_b200 import engine
    d = 6
    g = lq.parse("(1 + sum(i=1..d, x[i]))^(-(d+1))", d)
    counts = lq.axis_counts(lq.korobov_vector(4, 4**d + 1, d))
    plan = engine.linform_plan(g, counts)
    assert plan.ok and plan.wts is None
    ins, p = plan.program_struct()   # ins backs p's instruction pointer
    got = snippet["level_collapse_mean"](p, plan.m, plan.n, plan.h, plan.m0)
    assert got == engine.mdi_linform_mean(plan)
    assert abs(got - lq.mdi_lr(g, d, 4, 4**d + 1)) <= 1e-12 * got   # the grid mean is mdi_lr's value
