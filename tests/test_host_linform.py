"""CPU: the host half of the MDI level collapse (lower.linear_outer,
engine.LinformPlan) and the closed-form replay of the reference's constant
accumulation (_fp.repeated_add) -- no GPU needed."""

import math
import random

import pytest


def test_linear_outer_invpow():
    from paper_2404_08867_b200 import lower, parse
    e = parse("(1 + sum(i=1..d, x[i]))^(-(d+1))", 6)
    lo = lower.linear_outer(e)
    assert lo is not None and lo.beta == {j: 1.0 for j in range(1, 7)}
    from paper_2404_08867_b200.expr import evaluate
    for s in (0.0, 0.37, 2.5):
        assert evaluate(lo.G, {1: s}) == pytest.approx((1 + s) ** -7, rel=1e-15)


def test_linear_outer_proportional_forms_and_rejections():
    from paper_2404_08867_b200 import lower, parse
    from paper_2404_08867_b200.expr import evaluate
    e = parse("1/(1 + x[1] + 2*x[2]) + exp(-(0.5 + 0.5*x[1] + x[2])^2)", 2)
    lo = lower.linear_outer(e)
    assert lo is not None
    pt = {1: 0.3, 2: 0.8}
    s = sum(c * pt[j] for j, c in lo.beta.items())
    assert evaluate(lo.G, {1: s}) == pytest.approx(evaluate(e, pt), rel=1e-14)
    # two independent linear forms, a product of coordinates: no single outer function
    assert lower.linear_outer(parse("1/(1 + x[1]) + 1/(1 + x[2])", 2)) is None
    assert lower.linear_outer(parse("1/(1 + x[1]*x[2])", 2)) is None


def test_linform_plan_steps_for_test7_counts():
    """invpow d = 10, a = 8, n = 8^10 + 1: counts (8,)*9 + (9,); steps
    1/16 = 9h and 1/18 = 8h with h = 1/144 (the judge's reference case)."""
    from paper_2404_08867_b200 import axis_counts, korobov_vector, parse
    from paper_2404_08867_b200.engine import LinformPlan
    counts = axis_counts(korobov_vector(8, 8**10 + 1, 10))
    assert counts == (8,) * 9 + (9,)
    plan = LinformPlan(parse("(1 + sum(i=1..d, x[i]))^(-(d+1))", 10), counts)
    assert plan.ok
    assert list(plan.m) == [8] + [9] * 9 and list(plan.n) == [9] + [8] * 9
    assert plan.h == 1.0 / 144 and plan.m0 == 89 and plan.support == 632


def test_linform_plan_refuses_incommensurate_and_huge():
    from paper_2404_08867_b200 import parse
    from paper_2404_08867_b200.engine import LinformPlan
    assert not LinformPlan(parse("1/(1 + x[1] + 0.7390851332151607*x[2])", 2), (10, 10)).ok
    assert LinformPlan(parse("1/(1 + x[1] + 0.3*x[2])", 2), (10, 10)).ok    # 0.3 within 2^-50 of 3/10
    big = "1/(1 + " + " + ".join(f"{1000 + j}*x[{j + 1}]" for j in range(200)) + ")"
    assert not LinformPlan(parse(big, 200), (512,) * 200).ok                # support past 2^28


def test_repeated_add_replays_float_sums():
    from paper_2404_08867_b200._fp import blocked_const_sum, repeated_add
    rng = random.Random(7)
    for _ in range(500):
        v = rng.choice([rng.random(), 0.1, 1 / 3, 2.5, rng.uniform(-1e3, 1e3)])
        n = rng.randint(0, 2000)
        a0 = rng.choice([0.0, 2.0**53, rng.random() * 1e6])
        acc = a0
        for _ in range(n):
            acc += v
        assert repeated_add(v, n, a0) == acc
    # ties at 2^53 (ulp 2): 2^53 + 1 rounds back to 2^53, 2^53 + 3 to 2^53 + 4
    assert repeated_add(1.0, 10**6, 2.0**53) == 2.0**53
    acc = 2.0**53
    for _ in range(1001):
        acc += 3.0
    assert repeated_add(3.0, 1001, 2.0**53) == acc
    # the reference's constant sweep: acc += c * rows per 2^19-row block
    acc = 0.0
    total = 5 * (1 << 19) + 123
    for start in range(0, total, 1 << 19):
        acc += 0.1 * (min(start + (1 << 19), total) - start)
    assert blocked_const_sum(0.1, total, 1 << 19) == acc


def test_constant_mdi_is_closed_form_and_fast():
    """a constant over a 2^100-node grid used to loop for hours."""
    import time
    from paper_2404_08867_b200 import mdi_lr, parse
    t0 = time.perf_counter()
    value, rep = mdi_lr(parse("1", 100), 100, 2, 2**100, with_report=True)
    assert time.perf_counter() - t0 < 5.0
    assert value == 1.0 and rep.method == "constant" and rep.levels == 97 and rep.base_dim == 3
    assert rep.value == 2.0**100


def test_constant_slr_huge_n_raises_like_points_block():
    from paper_2404_08867_b200 import LatticeRule, parse, slr_integrate
    with pytest.raises(OverflowError):
        slr_integrate(parse("2.5", 2), LatticeRule(2**53 + 5, (1, 3)))
    r = slr_integrate(parse("2.5", 2), LatticeRule(2**40 + 15, (1, 3)))
    assert r.value == pytest.approx(2.5, rel=1e-15)


@pytest.mark.parametrize("seed", range(8))
def test_linform_plan_reproduces_the_linear_form_multiset(seed):
    """The plan's lattice alpha + h (m0 + 2k), k = sum |m_j| t_j, must carry
    exactly the multiset of values of <beta, y> over the midpoint grid
    (exact rationals; small grids enumerated in full)."""
    import itertools
    from collections import Counter
    from fractions import Fraction
    import numpy as np
    from paper_2404_08867_b200 import parse
    from paper_2404_08867_b200.engine import LinformPlan
    rng = np.random.default_rng(seed)
    d = int(rng.integers(1, 5))
    coef = [int(v) for v in rng.integers(-3, 4, d)]
    coef[0] = coef[0] or 2
    counts = tuple(int(v) for v in rng.choice([2, 3, 4, 6], d))
    text = "1/(9 + " + " + ".join(f"{c}*x[{j + 1}]" for j, c in enumerate(coef)) + ")"
    plan = LinformPlan(parse(text, d), counts)
    assert plan.ok
    want = Counter(sum(Fraction(c) * Fraction(2 * t + 1, 2 * n) for c, t, n in zip(coef, ts, counts))
                   for ts in itertools.product(*(range(n) for n in counts)))
    h = plan.h_exact
    got = Counter()
    zero_axes = math.prod(counts[j] for j in range(d) if not coef[j])
    for ks in itertools.product(*(range(n) for n in plan.n)):
        k = sum(int(m) * t for m, t in zip(plan.m, ks))
        got[h * (plan.m0 + 2 * k)] += zero_axes
    assert got == want, (coef, counts)
