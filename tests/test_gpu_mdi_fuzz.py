"""GPU: MDI-LR of random integrands on grids small enough for the direct
sweep.  Whatever branch mdi_sum picks -- separable cluster sums, core factors,
the level collapse of one linear form, unused-axis sub-grids, the direct sweep
-- the value must equal implr_integrate's direct sweep of the same grid
(mdi.py:104-136 vs 139-192: the reference pins the two to 1e-12,
tests/test_acceptance.py:52-71)."""

import math
import random

import pytest

pytestmark = pytest.mark.gpu


def _random_text(rng, d):
    def var():
        return f"x[{rng.randint(1, d)}]"

    def lin():
        k = rng.randint(1, d)
        return " + ".join(f"{rng.choice([1, 2, -1, 0.5, 0.25])}*{var()}" for _ in range(k))

    def atom(depth):
        r = rng.random()
        if depth > 2 or r < 0.3:
            return rng.choice([var(), f"({lin()})", repr(round(rng.uniform(0.1, 2.0), 3))])
        if r < 0.5:
            return f"exp({rng.choice([-1, 1]) * 0.5}*({atom(depth + 1)}))"
        if r < 0.6:
            return f"cos({atom(depth + 1)})"
        if r < 0.75:
            return f"(2 + {lin()})^({rng.choice([-1, -2, 2, 3])})"
        if r < 0.9:
            return f"{atom(depth + 1)}*{atom(depth + 1)}"
        return f"(1/(3 + ({atom(depth + 1)})^2))"

    return " + ".join(atom(0) for _ in range(rng.randint(1, 3)))


@pytest.mark.parametrize("seed", range(60))
def test_mdi_equals_direct_sweep_on_random_integrands(seed):
    import paper_2404_08867_b200 as lq
    rng = random.Random(seed)
    d = rng.randint(2, 6)
    a = rng.randint(2, 5 if d < 6 else 3)
    n = a**d + rng.choice([0, 1, 3])
    text = _random_text(rng, d)
    f = lq.parse(text, d)
    if not lq.free_vars(f):
        return
    value, rep = lq.mdi_lr(f, d, a, n, with_report=True)
    direct = lq.implr_integrate(f, d, a, n).value
    assert math.isfinite(direct)
    assert value == direct or math.isclose(value, direct, rel_tol=1e-10, abs_tol=1e-13), \
        (text, d, a, n, rep.method, value, direct)
