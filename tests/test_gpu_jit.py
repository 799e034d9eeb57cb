"""GPU: NVRTC-compiled integrands (jit.py) agree with the bytecode
interpreter and with the reference's golden values."""

import math
import os

import numpy as np
import pytest

from conftest import unhex

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lq():
    import paper_2404_08867_b200 as m
    return m


def _rule(lq, c):
    return lq.LatticeRule(int(c["n"]), tuple(int(v) for v in c["z"]))


def test_jit_plain_sums_match_interpreter_and_reference(lq, golden, monkeypatch):
    from paper_2404_08867_b200 import engine
    checked = 0
    for case in golden["slr"]:
        if case["value"] is None or case["tag"].startswith("cfg") or case["tag"] == "const_2p5":
            continue
        d = case["d"]
        f = lq.parse(case["text"], d)
        rule = _rule(lq, case)
        z = rule.z_reduced_array()
        monkeypatch.setenv("LQ_JIT", "0")
        engine._plain_cache.clear()
        interp = engine.plain_integrand(f, d, force_program=True)
        a = engine.lattice_sum(interp, rule.n, z)
        assert not interp.struct.prog.jit
        monkeypatch.setenv("LQ_JIT", "always")
        engine._plain_cache.clear()
        jitted = engine.plain_integrand(f, d, force_program=True)
        b = engine.lattice_sum(jitted, rule.n, z)
        assert jitted.struct.prog.jit, case["tag"]
        want = unhex(case["value"]) * rule.n
        assert abs(a - b) <= 1e-13 * max(abs(a), 1.0), case["tag"]
        assert abs(b - want) <= 1e-10 * max(abs(want), 1e-3 * rule.n), case["tag"]
        checked += 1
    assert checked >= 12


def test_jit_tensor_sums_match_reference(lq, golden, monkeypatch):
    monkeypatch.setenv("LQ_JIT", "always")
    checked = 0
    for case in golden["mdi"]:
        if "implr" not in case or not case["tag"].startswith(("acc01_expxy", "acc01_invpow", "acc01_sinsq")):
            continue
        f = lq.parse(case["text"], case["d"])
        got = lq.implr_integrate(f, case["d"], case["a"], int(case["n"])).value
        w = unhex(case["implr"])
        assert abs(got - w) <= 1e-12 * abs(w), case["tag"]
        checked += 1
    assert checked >= 30


def test_jit_wide_modulus(lq, monkeypatch):
    from paper_2404_08867_b200 import engine
    monkeypatch.setenv("LQ_JIT", "always")
    n = 2**40 + 15
    z = (1, 123456789013, 2**39 + 7)
    f = lq.parse("x[2]*exp(x[1]*x[3]) + sin(x[1]^2)", 3)
    pi = engine.plain_integrand(f, 3, force_program=True)
    lo = 2**35
    s = engine.lattice_sum(pi, n, np.asarray(z, dtype=np.uint64), lo, lo + 8192)
    assert pi.struct.prog.jit
    pts = np.array([[float((i * zj) % n) / n for zj in z] for i in range(lo, lo + 8192)])
    ref = float(np.sum(pts[:, 1] * np.exp(pts[:, 0] * pts[:, 2]) + np.sin(pts[:, 0] ** 2)))
    assert abs(s - ref) <= 1e-12 * abs(ref)


@pytest.mark.parametrize("n,lo,hi", [(2**40 + 15, 2**40 + 15 - 3000, 2**40 + 15 + 3001),   # wraps past n
                                     (2**40 + 15, 12345, 12345 + 70001),
                                     (2147483647, 2147483647 - 40003, 2147483647),
                                     (1000003, 7, 1000003)])
def test_jit_stepped_coordinates(lq, monkeypatch, n, lo, hi):
    # the JIT lattice kernel steps each used coordinate's residue from point
    # to point (r += z mod n) instead of forming i*z mod n: same coordinates as
    # the interpreter's per-point products, over unaligned sub-ranges and
    # ranges that cross i = n
    from paper_2404_08867_b200 import engine, jit
    d = 5
    f = lq.parse("x[2]*exp(x[1]*x[5]) + sin(x[1]^2) - x[4]^3", d)
    z = np.asarray([1, 123456789013 % n, (2**39 + 7) % n, 0, 977 % n], dtype=np.uint64)
    monkeypatch.setenv("LQ_JIT", "0")
    engine._plain_cache.clear()
    interp = engine.plain_integrand(f, d, force_program=True)
    a = engine.lattice_sum(interp, n, z, lo, hi)
    monkeypatch.setenv("LQ_JIT", "always")
    engine._plain_cache.clear()
    jitted = engine.plain_integrand(f, d, force_program=True)
    b = engine.lattice_sum(jitted, n, z, lo, hi)
    assert jitted.struct.prog.jit and "#define LQ_STEP" in jit.source_for(jitted.expr)
    assert abs(a - b) <= 1e-13 * max(abs(a), 1.0), (a, b)
    idx = np.arange(lo, hi, dtype=object) % n
    if len(idx) <= 80000:
        cols = [np.array([float(int(i) * int(zj) % n) / n for i in idx]) for zj in z]
        ref = float(np.sum(cols[1] * np.exp(cols[0] * cols[4]) + np.sin(cols[0] ** 2) - cols[3] ** 3))
        assert abs(b - ref) <= 1e-12 * abs(ref)


def test_jit_many_coordinates_unstepped(lq, monkeypatch):
    # past STEP_MAX_VARS used coordinates the kernel keeps per-point products
    from paper_2404_08867_b200 import engine, jit
    d = 30
    f = lq.parse("exp(-sum(i=1..d, x[i]^2)/7) + x[3]*x[30]", d)
    rule = lq.korobov_vector(4567, 2**35 + 3, d)
    monkeypatch.setenv("LQ_JIT", "0")
    engine._plain_cache.clear()
    a = engine.lattice_sum(engine.plain_integrand(f, d, force_program=True), rule.n, rule.z_reduced_array(), 0, 300000)
    monkeypatch.setenv("LQ_JIT", "always")
    engine._plain_cache.clear()
    pj = engine.plain_integrand(f, d, force_program=True)
    b = engine.lattice_sum(pj, rule.n, rule.z_reduced_array(), 0, 300000)
    assert pj.struct.prog.jit and "#define LQ_STEP" not in jit.source_for(pj.expr)
    assert abs(a - b) <= 1e-13 * abs(a)


def test_carried_state_across_tiles_lattice(lq, monkeypatch):
    # 2^25 indices: past one resident grid's worth of tiles (148 SMs x up to
    # 8 CTAs x 4096), so every thread carries its residues to further tiles;
    # the interpreter forms every coordinate by a modular product per point
    from paper_2404_08867_b200 import engine
    d = 4
    n = 2**41 + 21
    f = lq.parse("exp(-x[1]*x[2]) + cos(3*x[3] - x[4]^2)", d)
    z = np.asarray([1, 987654321987 % n, (2**40 + 3) % n, 55555], dtype=np.uint64)
    lo, hi = 12345, 12345 + (1 << 25)
    monkeypatch.setenv("LQ_JIT", "0")
    engine._plain_cache.clear()
    a = engine.lattice_sum(engine.plain_integrand(f, d, force_program=True), n, z, lo, hi)
    monkeypatch.setenv("LQ_JIT", "always")
    engine._plain_cache.clear()
    pj = engine.plain_integrand(f, d, force_program=True)
    b = engine.lattice_sum(pj, n, z, lo, hi)
    assert pj.struct.prog.jit
    assert abs(a - b) <= 1e-13 * abs(a), (a, b)


@pytest.mark.parametrize("jit_mode", ["0", "always"])
def test_carried_odometer_across_tiles_tensor(lq, monkeypatch, jit_mode):
    # a 2.1e7-node grid (more tiles than one resident grid holds): the carried
    # odometers of the interpreter and JIT tensor kernels against the oracle's
    # direct grid sum
    from oracle import np_oracle as orc
    from paper_2404_08867_b200 import engine
    from paper_2404_08867_b200.transform import AxisGridSet
    monkeypatch.setenv("LQ_JIT", jit_mode)
    text = "x[2]*exp(x[1]*x[2]) + sin(x[1] + x[3]^2)"
    counts = (277, 271, 281)
    f = lq.parse(text, 3)
    grids = AxisGridSet(None, counts, None, None, midpoint=True)
    got = engine.tensor_sum(f, grids)
    want = orc.direct_tensor_sum(text, orc.midpoint_nodes(list(counts)))
    assert abs(got - want) <= 1e-12 * abs(want), (got, want)
