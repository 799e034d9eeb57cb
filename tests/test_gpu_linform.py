"""GPU: MDI-LR level collapse for integrands that are functions of one
commensurate linear form (not separable) -- corpus invpow and relatives.  The
reference collapses their levels by like-term collection
(/root/reference/pkg/src/latquad/exprcore.py:139-169, 390-402;
mdi.py:152-165); lq_mdi_linform convolves the distribution of the partial
linear form one direction per level on the device.

Pinned three ways: reference mdi_lr goldens (tests/golden/linform.json,
frozen by tests/golden/make_golden.py --only linform), the exact
rational-multiset oracle (oracle.np_oracle.linear_form_grid_mean_exact), and
the GPU direct tensor sweep on grids under the direct cap."""

import math
from fractions import Fraction

import numpy as np
import pytest

from conftest import load_golden, unhex

pytestmark = pytest.mark.gpu

LINFORM = load_golden("linform")


@pytest.mark.parametrize("case", LINFORM, ids=lambda c: c["tag"])
def test_linform_matches_reference_golden(case):
    import paper_2404_08867_b200 as lq
    f = lq.parse(case["text"], case["d"])
    value, rep = lq.mdi_lr(f, case["d"], case["a"], int(case["n"]), with_report=True)
    want = unhex(case["value"])
    assert rep.method == "linform", rep.method
    assert abs(value - want) <= 1e-10 * abs(want), (value, want)
    assert abs(rep.value - unhex(case["raw"])) <= 1e-10 * abs(unhex(case["raw"]))
    assert (rep.levels, rep.base_dim, rep.fallback) == (case["levels"], case["base_dim"], case["fallback"])


def _grid(counts):
    from paper_2404_08867_b200.transform import AxisGridSet
    return AxisGridSet(None, counts, None, None, midpoint=True)


def _invpow(d):
    return lambda s: (1.0 + s) ** -(d + 1)


@pytest.mark.parametrize("d,a", [(3, 5), (5, 4), (7, 3), (12, 8), (16, 8)])
def test_invpow_matches_exact_multiset_oracle(d, a):
    import paper_2404_08867_b200 as lq
    from oracle.np_oracle import linear_form_grid_mean_exact
    n = 1 + a**d
    counts = lq.axis_counts(lq.korobov_vector(a, n, d))
    f = lq.parse("(1 + sum(i=1..d, x[i]))^(-(d+1))", d)
    value, rep = lq.mdi_lr(f, d, a, n, with_report=True)
    assert rep.method == "linform"
    steps = [Fraction(1, c) for c in counts]
    if d <= 7:
        want = linear_form_grid_mean_exact(_invpow(d), steps, counts)
        assert abs(value - want) <= 1e-12 * want, (value, want)
    else:   # test7 rows past the reference's build-container budget: numpy pmf oracle
        from oracle.np_oracle import linear_form_grid_mean_np
        L = math.lcm(*(2 * c for c in counts))
        k = [L // (2 * c) for c in counts]
        want = linear_form_grid_mean_np(_invpow(d), k, counts, 0.0, 1.0 / L)
        assert abs(value - want) <= 1e-12 * want, (value, want)


@pytest.mark.parametrize("seed", range(6))
@pytest.mark.parametrize("force_global", ["1", "0"])
def test_random_commensurate_forms(seed, force_global, monkeypatch):
    """Integer coefficients of both signs, zero coefficients, unequal counts
    (powers of two);
    both the shared-memory and the global-memory level kernels."""
    monkeypatch.setenv("LQ_LINFORM_SMEM", force_global)
    import paper_2404_08867_b200 as lq
    from oracle.np_oracle import linear_form_grid_mean_np
    rng = np.random.default_rng(100 + seed)
    d = int(rng.integers(3, 9))
    coef = [int(v) for v in rng.integers(-4, 5, d)]
    coef[0] = coef[0] or 1
    # commensurate node spacings (powers of two, or the Korobov (N, ..., N, N')
    # shape): unrelated counts make the partial forms' values distinct, the
    # support outgrows the node budget and the direct sweep runs, as in the
    # reference, whose constants then do not coincide either
    counts = tuple(int(v) for v in rng.choice([4, 8, 16, 32], d))
    alpha = 2.0 + float(sum(abs(c) for c in coef))
    text = f"({alpha!r} + " + " + ".join(f"{c}*x[{j + 1}]" for j, c in enumerate(coef)) + ")^(-2)"
    f = lq.parse(text, d)
    rep = lq.mdi_sum(f, _grid(counts))
    assert rep.method == "linform"
    L = math.lcm(*(2 * c for c in counts))
    k = [c * (L // (2 * n)) for c, n in zip(coef, counts)]
    want = linear_form_grid_mean_np(lambda s: s**-2, k, counts, alpha, 1.0 / L) * math.prod(counts)
    assert abs(rep.value - want) <= 1e-12 * abs(want), (rep.value, want)


def test_large_support_global_path_equals_numpy_pmf():
    """Support past shared memory (K > 12800): d = 80 directions with steps 1..5."""
    import paper_2404_08867_b200 as lq
    from oracle.np_oracle import linear_form_grid_mean_np
    d, N = 80, 64
    coef = [1 + (j % 5) for j in range(d)]
    text = "1/(1 + " + " + ".join(f"{c}*x[{j + 1}]" for j, c in enumerate(coef)) + ")"
    f = lq.parse(text, d)
    rep = lq.mdi_sum(f, _grid((N,) * d))
    assert rep.method == "linform" and rep.clusters > 12800
    want = linear_form_grid_mean_np(lambda s: 1.0 / s, coef, (N,) * d, 1.0, 1.0 / (2 * N))
    mean = rep.value / float(N) ** d
    assert abs(mean - want) <= 1e-12 * want, (mean, want)


@pytest.mark.parametrize("text,d,a,n", [
    ("1/(1 + x[1] + 2*x[2] - x[3])", 3, 7, 7**3),
    ("exp(-abs(x[1] - x[2] + 0.1))", 2, 10, 101),
    ("(2 + x[1] - 3*x[2] + x[3] + x[4])^(-3) + sin(x[1] - 3*x[2] + x[3] + x[4])", 4, 6, 6**4 + 5),
])
def test_linform_equals_direct_sweep(text, d, a, n):
    import paper_2404_08867_b200 as lq
    f = lq.parse(text, d)
    value, rep = lq.mdi_lr(f, d, a, n, with_report=True)
    assert rep.method == "linform"
    direct = lq.implr_integrate(f, d, a, n).value
    assert abs(value - direct) <= 1e-12 * abs(direct), (value, direct)


@pytest.mark.parametrize("nshards", [2, 3, 5])
def test_sharded_tiles_sum_to_the_single_gpu_mean(nshards):
    import torch
    import paper_2404_08867_b200 as lq
    from paper_2404_08867_b200 import _native as N
    from paper_2404_08867_b200 import engine
    d, N_ = 100, 64
    text = "1/(1 + " + " + ".join(f"{1 + j % 7}*x[{j + 1}]" for j in range(d)) + ")^2"
    plan = engine.linform_plan(lq.parse(text, d), (N_,) * d)
    assert plan.ok and plan.tiles >= nshards
    single = engine.mdi_linform_mean(plan)
    acc = torch.zeros(plan.tiles, dtype=torch.float64, device="cuda")
    for s in range(nshards):
        part = torch.empty(plan.tiles, dtype=torch.float64, device="cuda")
        engine.mdi_linform_mean(plan, s, nshards, part.data_ptr())
        torch.cuda.synchronize()
        acc += part     # disjoint writers: exact
    import ctypes as C
    out = C.c_double()
    N.check(N.lib().lq_reduce_sum(N.ctx(), C.c_void_p(acc.data_ptr()), plan.tiles, C.byref(out)))
    assert out.value == single


SUBGRID = load_golden("subgrid")


@pytest.mark.parametrize("case", SUBGRID, ids=lambda c: c["tag"])
def test_cores_and_unused_axes_match_reference(case):
    """Integrands that are not separable axis by axis but whose levels the
    reference still collapses: a piece on <= 3 axes (core, swept over its own
    sub-grid) times separable factors, or -- past 3 axes -- a sweep of the used
    axes alone with the unused ones multiplied in."""
    import paper_2404_08867_b200 as lq
    f = lq.parse(case["text"], case["d"])
    value, rep = lq.mdi_lr(f, case["d"], case["a"], int(case["n"]), with_report=True)
    want = unhex(case["value"])
    assert rep.method == ("subgrid" if case["tag"] == "exp4_d8" else "cores"), rep.method
    assert abs(value - want) <= 1e-10 * abs(want), (value, want)
    assert (rep.levels, rep.base_dim, rep.fallback) == (case["levels"], case["base_dim"], case["fallback"])


def test_weighted_level_collapse_matches_reference():
    """Products of separable real weights and a function of one commensurate
    linear form (tests/golden/linform_w.json, frozen from the reference's
    mdi_lr): each level's nodes carry phi_j(y_t) in the distribution update
    (lq_mdi_linform_w), including grids past the direct cap (d = 10, 12),
    weights on an axis outside the form and mixed-sign steps; and sums whose
    terms collapse by different branches (method "terms"); and functions of
    two commensurate forms (their joint distribution, method "linform2")."""
    methods = set()
    import paper_2404_08867_b200 as lq
    from conftest import load_golden, unhex
    for c in load_golden("linform_w"):
        f = lq.parse(c["text"], c["d"])
        cfg = lq.MdiConfig(m=c.get("m", 1), order=c.get("order", "forward"))
        got, rep = lq.mdi_lr(f, c["d"], c["a"], c["n"], cfg=cfg, with_report=True)
        want = unhex(c["value"])
        # a weighted form whose non-splitting piece spans <= 3 axes takes the
        # separable combine with a core instead (same collapse, same value)
        assert rep.method in ("linform", "cores", "terms", "linform2"), (c["text"], rep.method)
        assert abs(got - want) <= 1e-10 * abs(want), (c["text"], c["d"], got, want)
        assert (rep.levels, rep.base_dim, rep.fallback) == (c["levels"], c["base_dim"], c["fallback"]), c["text"]
        methods.add(rep.method)
    assert {"linform", "terms", "linform2"} <= methods, methods
