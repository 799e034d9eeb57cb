"""GPU parity against golden vectors frozen from the reference
(tests/golden/make_golden.py).  Bar: coordinates bit-exact; estimates within
relative 1e-10 (north star, BASELINE.json)."""

import math

import numpy as np
import pytest

from conftest import unb64, unhex

pytestmark = pytest.mark.gpu

REL = 1e-10


@pytest.fixture(scope="module")
def lq():
    import paper_2404_08867_b200 as m
    from paper_2404_08867_b200 import _native
    _native.lib()
    return m


def _rule(lq, case):
    return lq.LatticeRule(int(case["n"]), tuple(int(c) for c in case["z"]))


def test_points_bit_exact(lq, golden):
    for case in golden["points"]:
        rule = _rule(lq, case)
        got = lq.points_block(rule, case["start"], case["stop"])
        want = unb64(case["data"], case["shape"])
        assert got.shape == want.shape, case["tag"]
        assert np.array_equal(got.view(np.uint64), want.view(np.uint64)), case["tag"]


def test_lattice_points_and_blocks(lq):
    r = lq.LatticeRule(101, (1, 40))
    blocks = list(lq.iter_point_blocks(r, block=64))
    assert len(blocks) > 1
    assert np.array_equal(np.vstack(blocks), lq.lattice_points(r))
    pts = lq.lattice_points(lq.LatticeRule(4, (1, 3)))
    assert np.array_equal(pts, np.array([[0, 0], [0.25, 0.75], [0.5, 0.5], [0.75, 0.25]]))
    with pytest.raises(OverflowError):
        lq.lattice_points(lq.LatticeRule(2**54, (1,)))


def test_points_random_exhaustive_small_n(lq):
    # every residue class of several small moduli, against numpy's IEEE division
    for n in (1, 2, 3, 7, 97, 1009, 65537):
        rule = lq.LatticeRule(n, (1,))
        got = lq.lattice_points(rule)[:, 0]
        want = np.arange(n, dtype=np.int64) / n
        assert np.array_equal(got, want), n


def test_points_random_large(lq):
    rng = np.random.default_rng(7)
    for _ in range(6):
        n = int(rng.integers(2**20, 2**53))
        z = tuple(int(v) for v in rng.integers(1, min(n, 2**31), 5))
        start = int(rng.integers(0, n - 4096))
        rule = lq.LatticeRule(n, z)
        got = lq.points_block(rule, start, start + 4096)
        j = np.arange(start, start + 4096, dtype=object)
        want = np.array([[float((int(i) * zj) % n) / n for zj in z] for i in j])
        assert np.array_equal(got, want), n


def test_slr_golden(lq, golden):
    for case in golden["slr"]:
        if case["value"] is None:
            continue
        d = case["d"]
        f = lq.parse(case["text"], d)
        rule = _rule(lq, case)
        got = lq.slr_integrate(f, rule).value
        want = unhex(case["value"])
        if abs(want) < 1e-8:
            assert abs(got - want) <= 1e-13, case["tag"]
        else:
            assert abs(got - want) <= REL * abs(want), (case["tag"], got, want)


def test_slr_cfg5_ranges(lq, golden):
    from paper_2404_08867_b200 import engine
    for case in golden["slr"]:
        if not case["tag"].startswith("cfg5_range"):
            continue
        rule = _rule(lq, case)
        pi = engine.plain_integrand(lq.parse(case["text"], case["d"]), case["d"])
        assert pi.kind == "lin_expabs"
        got = engine.lattice_sum(pi, rule.n, rule.z_reduced_array(), case["i_begin"], case["i_end"])
        want = unhex(case["range_sum"])
        assert abs(got - want) <= REL * abs(want), (case["tag"], got, want)


def test_slr_program_path_matches_family_path(lq, golden):
    # the generic bytecode kernel and the family kernels agree on every config
    from paper_2404_08867_b200 import engine
    for case in golden["slr"]:
        if not case["tag"].startswith("cfg") or case["value"] is None:
            continue
        d = case["d"]
        rule = _rule(lq, case)
        f = lq.parse(case["text"], d)
        fam = engine.plain_integrand(f, d)
        prog = engine.plain_integrand(f, d, force_program=True)
        a = engine.lattice_sum(fam, rule.n, rule.z_reduced_array())
        b = engine.lattice_sum(prog, rule.n, rule.z_reduced_array())
        assert abs(a - b) <= REL * abs(b), (case["tag"], a, b)


def test_mdi_golden(lq, golden):
    for case in golden["mdi"]:
        if "text" not in case:
            continue
        d, a, n = case["d"], case["a"], int(case["n"])
        f = lq.parse(case["text"], d)
        cfg = lq.MdiConfig(direct_cap=case["direct_cap"]) if "direct_cap" in case else None
        value, rep = lq.mdi_lr(f, d, a, n, cfg=cfg, with_report=True)
        raw = unhex(case["raw"])
        want = unhex(case["value"])
        if raw != 0.0 and math.isfinite(raw):
            assert abs(rep.value - raw) <= REL * abs(raw), (case["tag"], rep.value, raw)
        if want != 0.0:
            assert abs(value - want) <= REL * abs(want), (case["tag"], value, want)
        else:
            assert value == 0.0, case["tag"]
        if rep.method in ("separable", "cores", "linform", "subgrid"):
            # levels collapse (product form, one commensurate linear form, or
            # unused axes stripped in front of a sweep over the used ones)
            assert (rep.levels, rep.base_dim) == (case["levels"], case["base_dim"]), case["tag"]
            if rep.method != "separable":
                assert not case["fallback"], case["tag"]
        else:   # non-separable: the reference's full-grid fallback sweep (mdi.py:167-179)
            assert rep.method in ("direct", "constant"), case["tag"]
        if "implr" in case:
            got = lq.implr_integrate(f, d, a, n).value
            w = unhex(case["implr"])
            assert abs(got - w) <= 1e-12 * abs(w), (case["tag"], got, w)


def test_mdi_cfg4_log_raw(lq, golden):
    case = next(c for c in golden["mdi"] if c.get("tag") == "cfg4")
    f = lq.parse(case["text"], case["d"])
    value, rep = lq.mdi_lr(f, case["d"], case["a"], int(case["n"]), with_report=True)
    assert value == 0.0   # the reference underflows too
    assert abs(rep.log_raw - unhex(case["log_raw"])) <= 1e-10 * abs(unhex(case["log_raw"]))


def test_mdi_cap_refusal(lq, golden):
    from paper_2404_08867_b200.configs import make_config
    cfg = make_config(1)
    f = lq.parse(cfg.text, cfg.d)
    with pytest.raises(lq.GridCapError):
        lq.mdi_lr(f, cfg.d, cfg.mdi_a, cfg.mdi_n)
