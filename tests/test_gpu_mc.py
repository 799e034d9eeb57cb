"""GPU Monte Carlo (quad.mc_integrate, quad.py:79-93) against values frozen
from the reference: the device reproduces numpy's default_rng(seed) PCG64
stream, so the points are bit-identical and the means agree to summation-order
rounding."""

import ctypes as C
import math

import numpy as np
import pytest

from conftest import load_golden, unb64, unhex

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lq():
    import paper_2404_08867_b200 as m
    from paper_2404_08867_b200 import _native
    _native.lib()
    return m


def test_mc_values_match_reference(lq):
    for case in load_golden("mc"):
        f = lq.parse(case["text"], case["d"])
        r = lq.mc_integrate(f, case["d"], case["n"], seed=case["seed"], reference=1.0)
        want = unhex(case["value"])
        assert r.method == "mc" and r.seed == case["seed"] and r.points == case["n"]
        assert math.isclose(r.value, want, rel_tol=1e-12), (case["tag"], r.value, want)


def test_mc_points_bit_exact(lq):
    # a one-point "sum" of the coordinate program x[j] is the coordinate itself
    from paper_2404_08867_b200 import _native as N, engine
    for case in load_golden("mc"):
        d = case["d"]
        first = unb64(case["first_rows"], case["first_shape"])
        st = np.random.default_rng(case["seed"]).bit_generator.state["state"]
        m64 = (1 << 64) - 1
        state = np.array([st["state"] & m64, st["state"] >> 64], dtype=np.uint64)
        inc = np.array([st["inc"] & m64, st["inc"] >> 64], dtype=np.uint64)
        for j in range(d):
            prog = engine.tensor_program(lq.parse(f"x[{j + 1}]", d))
            ins = np.ascontiguousarray(prog.insn)
            p = N.Program(ins.ctypes.data, len(ins), prog.n_slots, prog.result, prog.n_vars, None)
            for i in range(first.shape[0]):
                out = C.c_double()
                N.check(N.lib().lq_mc_sum(N.ctx(), C.byref(p), d, case["n"], N.as_ptr(state), N.as_ptr(inc),
                                          i, i + 1, C.byref(out)))
                assert out.value == first[i, j], (case["tag"], i, j)


def test_mc_far_stream_offsets(lq):
    # points deep in the stream (jump-ahead by ~2^40 draws) against the oracle's jump
    from paper_2404_08867_b200 import _native as N, engine
    from oracle import np_oracle
    d, n, seed = 3, 1 << 40, 2024
    st = np.random.default_rng(seed).bit_generator.state["state"]
    m64 = (1 << 64) - 1
    state = np.array([st["state"] & m64, st["state"] >> 64], dtype=np.uint64)
    inc = np.array([st["inc"] & m64, st["inc"] >> 64], dtype=np.uint64)
    for j in range(d):
        prog = engine.tensor_program(lq.parse(f"x[{j + 1}]", d))
        ins = np.ascontiguousarray(prog.insn)
        p = N.Program(ins.ctypes.data, len(ins), prog.n_slots, prog.result, prog.n_vars, None)
        for i in (12345, (1 << 39) + 7, n - 1):
            out = C.c_double()
            N.check(N.lib().lq_mc_sum(N.ctx(), C.byref(p), d, n, N.as_ptr(state), N.as_ptr(inc), i, i + 1,
                                      C.byref(out)))
            assert out.value == np_oracle.pcg64_draw(st["state"], st["inc"], i * d + j), (i, j)


def test_mc_errors(lq):
    with pytest.raises(ValueError):
        lq.mc_integrate(lq.parse("x[1]", 1), 1, 0)
    r = lq.mc_integrate(lq.parse("2.5", 3), 3, 1000)
    assert r.value == 2.5


def test_mc_seed_determinism_and_three_sigma(lq):
    # the reference's own Monte-Carlo checks (tests/test_quad.py TestMonteCarlo)
    from paper_2404_08867_b200 import corpus
    f = corpus.corpus_expr("gaussian", 3)
    a = lq.mc_integrate(f, d=3, n=4096, seed=11)
    b = lq.mc_integrate(f, d=3, n=4096, seed=11)
    c = lq.mc_integrate(f, d=3, n=4096, seed=12)
    assert a.value == b.value and a.value != c.value
    r = lq.mc_integrate(lq.parse("x[1]", 1), d=1, n=10**6, seed=0)
    assert abs(r.value - 0.5) <= 3.0 * (1.0 / math.sqrt(12.0)) / 1e3
    r = lq.mc_integrate(corpus.corpus_expr("expsum", 3), d=3, n=10**4, seed=5, reference=1.0)
    assert r.rel_error == pytest.approx(abs(r.value - 1.0))


def test_mc_error_slope(lq):
    # acceptance check 10 of the reference: mean |error| ~ n^-1/2
    from paper_2404_08867_b200 import corpus
    f = corpus.corpus_expr("gaussian", 2)
    ref = corpus.reference_value("gaussian", 2)
    ns = [10**3, 10**4, 10**5]
    means = [np.mean([lq.mc_integrate(f, 2, n, seed=s, reference=ref).rel_error for s in range(16)]) for n in ns]
    slope = float(np.polyfit(np.log(ns), np.log(means), 1)[0])
    assert abs(slope + 0.5) <= 0.15, slope
