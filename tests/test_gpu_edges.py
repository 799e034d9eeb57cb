"""GPU: edge cases of the boundary -- empty/ragged ranges, tiny and maximal
moduli, the family/bytecode switch at n = 2^31, d beyond the parameter-space
table, negative point indices, constant and single-point rules."""

import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lq():
    import paper_2404_08867_b200 as m
    return m


def test_empty_and_single_point(lq):
    from paper_2404_08867_b200 import engine
    r = lq.LatticeRule(1, (1, 1, 1))
    f = lq.parse("exp(x[1] + 2*x[2] - x[3])", 3)
    assert lq.slr_integrate(f, r).value == 1.0          # the single point is the origin
    pi = engine.plain_integrand(f, 3)
    assert engine.lattice_sum(pi, 1009, np.array([1, 5, 7], dtype=np.uint64), 500, 500) == 0.0
    assert lq.points_block(lq.LatticeRule(7, (1, 3)), 5, 5).shape == (0, 2)


def test_ragged_ranges_add_up(lq):
    from paper_2404_08867_b200 import engine
    from paper_2404_08867_b200.configs import make_config
    cfg = make_config(2)
    rule = lq.korobov_vector(cfg.plain_a, cfg.plain_n, cfg.d)
    pi = engine.plain_integrand(lq.parse(cfg.text, cfg.d), cfg.d)
    z = rule.z_reduced_array()
    whole = engine.lattice_sum(pi, rule.n, z)
    cuts = [0, 1, 17, 4099, 6145, 9999, rule.n]
    parts = sum(engine.lattice_sum(pi, rule.n, z, a, b) for a, b in zip(cuts[:-1], cuts[1:]))
    assert abs(parts - whole) <= 1e-12 * abs(whole)


def test_negative_start_points(lq):
    from oracle import np_oracle as orc
    rule = lq.LatticeRule(101, (1, 40, 77))
    got = lq.points_block(rule, -5, 7)
    want = orc.points_block(101, (1, 40, 77), -5, 7)      # numpy's % wraps like the reference
    assert np.array_equal(got, want)


@pytest.mark.parametrize("n", [2**31 - 1, 2**31, 2**31 + 11])
def test_modulus_boundary_family_vs_bytecode(lq, n):
    from paper_2404_08867_b200 import engine
    d = 6
    text = "exp(-abs(0.3*x[1] - 0.2*x[2] + 0.5*x[3] - 0.1*x[4] + 0.25*x[5] - 0.4*x[6] + 0.05))"
    f = lq.parse(text, d)
    z = np.array([1, 1234567, 987654321 % n, 5, 2**30 + 3, 77], dtype=np.uint64)
    fam = engine.plain_integrand(f, d)
    prog = engine.plain_integrand(f, d, force_program=True)
    lo, hi = n - 300_000, n                                    # the top of the index range
    a = engine.lattice_sum(fam, n, z, lo, hi)
    b = engine.lattice_sum(prog, n, z, lo, hi)
    assert abs(a - b) <= 1e-12 * abs(b)
    from oracle import np_oracle as orc
    want = orc.slr_sum(text, n, [int(v) for v in z], lo, lo + 4096)
    got = engine.lattice_sum(fam, n, z, lo, lo + 4096)
    assert abs(got - want) <= 1e-12 * abs(want)


def test_wide_modulus_points_and_sum(lq):
    from oracle import np_oracle as orc
    from paper_2404_08867_b200 import engine
    n = 2**40 + 15
    z = (1, 123456789013, 2**39 + 7)
    rule = lq.LatticeRule(n, z)
    got = lq.points_block(rule, 2**35, 2**35 + 64)
    j = range(2**35, 2**35 + 64)
    want = np.array([[float((i * zj) % n) / n for zj in z] for i in j])
    assert np.array_equal(got, want)
    f = lq.parse("cos(x[1] + 2*x[2] - x[3])", 3)
    pi = engine.plain_integrand(f, 3)
    s = engine.lattice_sum(pi, n, rule.z_reduced_array(), 2**35, 2**35 + 8192)
    # exact residues in Python ints: numpy's int64 j*z would wrap here (as the
    # reference's points_block silently does for n past ~3e9)
    pts = np.array([[float((i * zj) % n) / n for zj in z] for i in range(2**35, 2**35 + 8192)])
    ref = float(np.sum(np.cos(pts[:, 0] + 2 * pts[:, 1] - pts[:, 2])))
    assert abs(s - ref) <= 1e-12 * abs(ref)


def test_dimension_beyond_parameter_table(lq):
    # d > 1000 takes the global-memory table; d = 1500 lin and quad families vs bytecode
    from paper_2404_08867_b200 import engine
    d, n, a = 1500, 100_003, 7919
    rng = np.random.default_rng(5)
    c = rng.uniform(0, 0.02, d)
    w = rng.uniform(0, 1, d)
    rule = lq.korobov_vector(a, n, d)
    z = rule.z_reduced_array()
    for text in ("exp(-abs(" + " + ".join(f"{float(cj)!r}*(x[{j + 1}]-{float(wj)!r})" for j, (cj, wj) in enumerate(zip(c, w))) + "))",
                 "exp(-(" + " + ".join(f"{float(cj)!r}*(x[{j + 1}]-{float(wj)!r})^2" for j, (cj, wj) in enumerate(zip(c, w))) + "))"):
        f = lq.parse(text, d)
        fam = engine.plain_integrand(f, d)
        assert fam.kind in ("lin_expabs", "quad_exp")
        prog = engine.plain_integrand(f, d, force_program=True)
        x = engine.lattice_sum(fam, n, z)
        y = engine.lattice_sum(prog, n, z)
        assert abs(x - y) <= 1e-11 * abs(y), fam.kind


def test_tensor_sum_custom_grids_and_cap(lq):
    from paper_2404_08867_b200.transform import AxisGridSet
    g = lq.parse("x[1]^2 + x[1]*x[2] + x[2]^2", 2)
    third = (0.0, 1.0 / 3.0, 2.0 / 3.0)
    grids = AxisGridSet((third, third), (3, 3), 0, (1, 1))
    want = sum(a * a + a * b + b * b for a in third for b in third)
    assert lq.mdi_sum(g, grids).value == pytest.approx(want, rel=1e-14)
    assert lq.direct_tensor_sum(lq.parse("x[1]^2", 1), AxisGridSet(((0.0, 0.25, 0.5, 0.75),), (4,), 0, (1,))) \
        == pytest.approx(0.875, rel=1e-15)
    with pytest.raises(lq.GridCapError):
        lq.direct_tensor_sum(lq.parse("exp(-x[1]*x[2])", 4), lq.midpoint_grids(lq.korobov_vector(4, 256, 4)), cap=100)


def test_mdi_policies(lq):
    f = lq.parse("(1 + sum(i=1..d, x[i]))^(-(d+1))", 5)
    rep = lq.mdi_sum(f, lq.midpoint_grids(lq.korobov_vector(3, 3**5, 5)), lq.MdiConfig(budget=1))
    assert rep.fallback and rep.value == lq.direct_tensor_sum(f, lq.midpoint_grids(lq.korobov_vector(3, 3**5, 5)))
    with pytest.raises(lq.BudgetExceededError):
        lq.mdi_sum(f, lq.midpoint_grids(lq.korobov_vector(3, 3**5, 5)), lq.MdiConfig(budget=1, fallback="error"))
    with pytest.raises(ValueError):
        lq.mdi_sum(lq.parse("x[3]", 3), lq.midpoint_grids(lq.korobov_vector(2, 4, 2)))
    for d, a, n in ((2, 10, 101), (4, 3, 81), (6, 2, 64)):
        assert lq.mdi_lr(lq.parse("1", d), d, a, n) == 1.0
    g = lq.parse("exp(sum(i=1..d, (-1)^(i+1)*x[i]))", 7)
    grids = lq.AxisGridSet(((0.25, 0.75),) * 7, (2,) * 7, 0, (1,) * 7)
    for m in (1, 2, 3):
        rep = lq.mdi_sum(g, grids, lq.MdiConfig(m=m))
        assert rep.levels == math.ceil((7 - rep.base_dim) / m) and 1 <= rep.base_dim <= 3


def test_mdi_m_order_invariance_and_huge_grid(lq):
    # the reference's TestMdiSum.test_m_and_order_invariance / test_huge_grid_normalization
    from paper_2404_08867_b200 import corpus
    f = corpus.corpus_expr("sinsq", 6)
    grids = lq.midpoint_grids(lq.korobov_vector(3, 3**6, 6))
    base = lq.mdi_sum(f, grids, lq.MdiConfig(m=1)).value
    for m in (1, 2, 3):
        for order in ("forward", "reverse"):
            got = lq.mdi_sum(f, grids, lq.MdiConfig(m=m, order=order)).value
            assert got == pytest.approx(base, rel=1e-12)
    g = corpus.corpus_expr("expalt", 20)
    got = lq.mdi_lr(g, 20, 8, 8**20)
    ref = corpus.reference_value("expalt", 20)
    assert math.isfinite(got) and abs(got - ref) / abs(ref) < 2e-2
