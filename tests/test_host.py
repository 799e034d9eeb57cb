"""CPU: host-side logic of the drop-in (parser, lowering, bookkeeping, ABI)."""

import ctypes
import math
import os
import re

import numpy as np
import pytest
from hypothesis import given, settings, strategies as st

import paper_2404_08867_b200 as lq
from paper_2404_08867_b200 import expr as E
from paper_2404_08867_b200 import lower as L
from paper_2404_08867_b200.configs import make_config
from paper_2404_08867_b200.mdi import _det_a, _level_plan, _normalize
from paper_2404_08867_b200.transform import axis_counts, midpoint_grids

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


# ---------------------------------------------------------------- parser

def test_parser_quirks_match_reference_grammar():
    x = E.var(1)
    assert E.evaluate(lq.parse("-x[1]^2", 1), {1: 3.0}) == 9.0          # (-a)^k, exprcore.py:591-603
    assert E.evaluate(lq.parse("x[1]/4", 1), {1: 2.0}) == 0.5
    assert E.evaluate(lq.parse("2/(1+x[1])", 1), {1: 1.0}) == 1.0
    assert E.evaluate(lq.parse("sum(i=1..d, i*x[i])", 3), {1: 1, 2: 1, 3: 1}) == 6.0
    assert E.evaluate(lq.parse("prod(i=1..d, x[i]^(i))", 3), {1: 2, 2: 2, 3: 2}) == 64.0
    assert E.evaluate(lq.parse("exp(sum(i=1..d, (-1)^(i+1)*x[i]))", 2), {1: 1.0, 2: 1.0}) == 1.0
    assert E.evaluate(lq.parse("2*pi + e", 1), {}) == 2 * math.pi + math.e
    assert E.evaluate(lq.parse("abs(x[1]-1)", 1), {1: 0.25}) == 0.75     # extension
    for bad in ("x[0]", "x[3]", "foo(1)", "x[1]/x[2]", "(1", "1 $ 2", "x[1]/0"):
        with pytest.raises(lq.ParseError):
            lq.parse(bad, 2)


def test_repr_float_literals_round_trip():
    cfg = make_config(2)
    f = lq.parse(cfg.text, cfg.d)
    fam = L.recognize_plain(f, cfg.d)
    assert fam.kind == "lin_sincos"
    assert np.array_equal(fam.beta, np.asarray(cfg.c))


def test_reference_expr_adapter_duck_typing():
    class R:   # minimal stand-in for a latquad Expr node (exprcore.py:80-91)
        def __init__(self, kind, value=0.0, index=0, children=()):
            self.kind, self.value, self.index, self.children = kind, value, index, children
    x1, x2 = R("var", index=1), R("var", index=2)
    s = R("sum", 0.5, 0, ((x1, 2.0), (x2, -1.0)))
    e = R("exp", children=(s,))
    p = R("prod", 3.0, 0, (e, R("pow", 0.0, -1, (x2,))))
    got = E.as_expr(p)
    assert E.evaluate(got, {1: 0.3, 2: 0.7}) == pytest.approx(3.0 * math.exp(0.5 + 0.6 - 0.7) / 0.7, rel=1e-15)


# ------------------------------------------------------------- lowering

@pytest.mark.parametrize("cid,kind", [(1, "lin_exp"), (2, "lin_sincos"), (3, "quad_exp"), (5, "lin_expabs")])
def test_config_families_recognised(cid, kind):
    cfg = make_config(cid)
    fam = L.recognize_plain(lq.parse(cfg.text, cfg.d), cfg.d)
    assert fam is not None and fam.kind == kind


def _family_value(fam, x):
    if fam.kind == "lin_exp":
        return fam.K * math.exp(fam.alpha + float(fam.beta @ x))
    if fam.kind == "lin_sincos":
        L_ = float(fam.beta @ x)
        return fam.C0 + fam.A * math.sin(L_) + fam.B * math.cos(L_)
    if fam.kind == "lin_expabs":
        return fam.K * math.exp(fam.kappa * abs(fam.alpha + float(fam.beta @ x)))
    return fam.K * math.exp(fam.alpha + float(fam.beta @ x) + float(fam.gamma @ (x * x)))


@pytest.mark.parametrize("cid", [1, 2, 3, 5])
def test_family_parameters_reproduce_the_integrand(cid):
    cfg = make_config(cid)
    f = lq.parse(cfg.text, cfg.d)
    fam = L.recognize_plain(f, cfg.d)
    rng = np.random.default_rng(cid)
    for _ in range(5):
        x = rng.uniform(0, 1, cfg.d)
        want = E.evaluate(f, {j + 1: x[j] for j in range(cfg.d)})
        assert _family_value(fam, x) == pytest.approx(want, rel=1e-12, abs=1e-14)


def _run_bytecode(prog, xs):
    """Python interpreter of the liblq bytecode (mirror of lq_device.cuh::run_program)."""
    slot = [0.0] * prog.n_slots
    for op, a, b, n, c in prog.insn.tolist():
        if op == L.OP_CONST or op == L.OP_ACC_INIT:
            slot[a] = c
        elif op == L.OP_VAR:
            slot[a] = xs[b]
        elif op == L.OP_ACC_ADD:
            slot[a] = slot[a] + c * slot[b]
        elif op == L.OP_ACC_ADDVAR:
            slot[a] = slot[a] + c * xs[b]
        elif op == L.OP_ACC_MUL:
            slot[a] = slot[a] * slot[b]
        elif op == L.OP_POW:
            slot[a] = slot[b] ** n
        elif op == L.OP_RPOW:
            slot[a] = 1.0 / (slot[b] ** n)
        else:
            slot[a] = {L.OP_EXP: math.exp, L.OP_SIN: math.sin, L.OP_COS: math.cos, L.OP_ABS: abs}[op](slot[b])
    return slot[prog.result]


CORPUS_LIKE = [
    ("x[2]*exp(x[1]*x[2])/(e-2)", 2), ("sin(2*pi + sum(i=1..d, x[i]^2))", 4),
    ("exp(sum(i=1..d, x[i])) / (e-1)^d", 3), ("0.3989422804014327*exp(-sum(i=1..d, x[i]^2)/2)", 5),
    ("prod(i=1..d, 1/(0.81 + (x[i]-0.6)^2))", 4), ("(1 + sum(i=1..d, x[i]))^(-(d+1))", 3),
    ("cos(2*pi + sum(i=1..d, 2*x[i]))", 6), ("x[1]^3*x[2] - 0.5*x[3]^2 + x[1]*x[2]*x[3] + 0.25", 3),
    ("exp(-abs(0.3*x[1] - 0.2*x[2] + 0.1))", 2), ("(x[1] + x[2])^2 * (x[1] - x[2])^-2", 2),
]


@pytest.mark.parametrize("text,d", CORPUS_LIKE)
def test_bytecode_matches_host_evaluation(text, d):
    f = lq.parse(text, d)
    prog = L.compile_program(f)
    rng = np.random.default_rng(len(text))
    for _ in range(10):
        x = rng.uniform(0.05, 0.95, d)
        want = E.evaluate(f, {j + 1: x[j] for j in range(d)})
        assert _run_bytecode(prog, list(x)) == pytest.approx(want, rel=1e-13, abs=1e-300)
    assert prog.n_slots <= L.MAX_SLOTS


def _sep_eval(terms, x):
    tot = 0j
    for t in terms:
        v = complex(t.coef)
        for axes, fc in t.factors.items():
            pt = {ax: x[ax - 1] for ax in axes}
            R = E.evaluate(fc.R, pt) if fc.R is not None else 1.0
            P = E.evaluate(fc.P, pt) if fc.P is not None else 0.0
            v *= R * complex(math.cos(P), math.sin(P))
        tot += v
    return tot


@pytest.mark.parametrize("text,d", [t for t in CORPUS_LIKE if "abs" not in t[0] and "^(-(d+1))" not in t[0]
                                    and "exp(x[1]*x[2])" not in t[0] and "^-2" not in t[0]])
def test_separation_is_exact(text, d):
    f = lq.parse(text, d)
    terms = L.separate(f)
    assert terms is not None
    rng = np.random.default_rng(d)
    for _ in range(6):
        x = rng.uniform(0, 1, d)
        want = E.evaluate(f, {j + 1: x[j] for j in range(d)})
        got = _sep_eval(terms, x)
        assert abs(got.imag) <= 1e-12 * max(1.0, abs(want))
        assert got.real == pytest.approx(want, rel=1e-12, abs=1e-12)


def test_non_separable_detected():
    for text, d in [("x[2]*exp(x[1]*x[2])", 2), ("(1 + x[1] + x[2])^(-3)", 2), ("exp(-abs(x[1] - x[2]))", 2)]:
        assert L.separate(lq.parse(text, d)) is None


@pytest.mark.parametrize("text,d,cores", [
    ("exp(x[1]*x[2])*prod(i=3..d, 1/(1 + x[i]^2))", 6, {(1, 2)}),
    ("exp(x[1]*x[2] + x[3] + sum(i=4..d, 0.5*x[i]))", 7, {(1, 2)}),
    ("cos(x[1]*x[5] + x[2]) + x[3]*x[4]", 5, {(1, 5)}),
    ("(1 + x[1] + x[2] + x[3])^(-3)*exp(x[4]) + sin(x[5])", 5, {(1, 2, 3)}),
    ("x[2]*exp(x[1]*x[2])/(e-2)*prod(i=3..d, x[i])", 4, {(1, 2)}),
])
def test_separation_with_cores_is_exact(text, d, cores):
    """max_axes = 3: non-splitting pieces on <= 3 coordinates become core
    factors; the factorisation must still reproduce f exactly."""
    f = lq.parse(text, d)
    assert L.separate(f) is None
    terms = L.separate(f, max_axes=3)
    assert terms is not None
    seen = {key for t in terms for key in t.factors if len(key) > 1}
    assert seen == cores, seen
    rng = np.random.default_rng(d)
    for _ in range(6):
        x = rng.uniform(0, 1, d)
        want = E.evaluate(f, {j + 1: x[j] for j in range(d)})
        got = _sep_eval(terms, x)
        assert abs(got.imag) <= 1e-12 * max(1.0, abs(want))
        assert got.real == pytest.approx(want, rel=1e-12, abs=1e-12)


def test_cores_larger_than_three_axes_are_refused():
    f = lq.parse("exp(x[1]*x[2]*x[3]*x[4])*x[5]", 5)
    assert L.separate(f, max_axes=3) is None


_coef = st.floats(min_value=-2, max_value=2, allow_nan=False)


@given(st.lists(st.tuples(st.integers(1, 4), st.integers(1, 3), _coef), min_size=1, max_size=6), _coef)
@settings(max_examples=40, deadline=None)
def test_separation_random_polynomials(monos, c0):
    pairs = [(c, E.power(E.var(i), k)) for i, k, c in monos]
    f = E.add(pairs, c0)
    terms = L.separate(f)
    assert terms is not None
    x = np.linspace(0.1, 0.9, 4)
    want = E.evaluate(f, {j + 1: x[j] for j in range(4)})
    assert _sep_eval(terms, x).real == pytest.approx(want, rel=1e-12, abs=1e-12)


# ---------------------------------------------------- rules and bookkeeping

def test_lattice_rule_validation_mirrors_reference():
    with pytest.raises(ValueError):
        lq.LatticeRule(0, (1,))
    with pytest.raises(ValueError):
        lq.LatticeRule(5, ())
    with pytest.raises(ValueError):
        lq.LatticeRule(5, (1, 0))
    r = lq.korobov_vector(7, 81, 3)
    assert r.z == (1, 7, 49) and r.z_reduced == (1, 7, 49)
    big = lq.korobov_vector(10, 101, 3)
    assert big.z == (1, 10, 100) and not big.is_grid_type
    assert lq.LatticeRule(4, (1, 2)).is_grid_type
    assert len({lq.LatticeRule(8, (1, 3)), lq.LatticeRule(8, (1, 3))}) == 1
    with pytest.raises(ValueError):
        lq.korobov_vector(0, 11, 2)
    with pytest.raises(ValueError):
        lq.korobov_vector(11, 11, 2)
    cfg = make_config(5)
    rule = lq.korobov_vector(cfg.plain_a, cfg.plain_n, cfg.d)
    assert rule.z_reduced == tuple(c % rule.n for c in rule.z[:0]) + cfg.plain_z()


def test_axis_counts_closed_form_equals_lcm_form():
    for a, n, d in [(3, 81, 4), (10, 1 + 10**10, 10), (478, 1009, 8), (64, 64**100, 100), (1, 11, 4)]:
        kor = lq.korobov_vector(a, n, d)
        plain = lq.LatticeRule(n, kor.z)
        assert axis_counts(kor) == axis_counts(plain)
    assert midpoint_grids(lq.korobov_vector(2, 8, 3)).nodes == ((0.25, 0.75),) * 2 + ((0.25, 0.75),)


def test_level_plan_matches_reference_reports(golden):
    for case in golden["mdi"]:
        if "levels" not in case:
            continue
        levels, base = _level_plan(case["d"], lq.MdiConfig())
        assert (levels, len(base)) == (case["levels"], case["base_dim"]), case["tag"]


def test_mdiconfig_validation():
    for kw in ({"m": 0}, {"m": 4}, {"budget": 0}, {"order": "sideways"}, {"fallback": "retry"}):
        with pytest.raises(ValueError):
            lq.MdiConfig(**kw)
    cfg = lq.MdiConfig()
    assert cfg.m == 1 and cfg.order == "forward" and cfg.fallback == "numeric"


def test_det_a_and_normalize(golden):
    for case in golden["mdi"]:
        if case.get("det_a") is None:
            continue
        rule = lq.korobov_vector(case["a"], int(case["n"]), case["d"])
        assert _det_a(rule) == float.fromhex(case["det_a"]), case["tag"]
        counts = axis_counts(rule)
        assert _normalize(float.fromhex(case["raw"]), counts) == float.fromhex(case["value"])


def test_quadrature_result_validation():
    with pytest.raises(ValueError):
        lq.QuadratureResult(method="slr", value=1.0, points=0, d=1, n=1)
    with pytest.raises(ValueError):
        lq.QuadratureResult(method="slr", value=1.0, points=1, d=1, n=1, rel_error=-0.1)


# -------------------------------------------------------------- C ABI

def test_library_exports_every_declared_symbol():
    from paper_2404_08867_b200 import _native
    if not os.path.exists(_native.LIB_PATH):
        pytest.skip("liblq.so not built")
    header = open(os.path.join(REPO, "include", "lq.h")).read()
    names = set(re.findall(r"^\s*(?:int|int64_t|const char\*)\s+(lq_\w+)\s*\(", header, re.M))
    assert len(names) >= 18
    lib = ctypes.CDLL(_native.LIB_PATH)
    for name in sorted(names):
        assert hasattr(lib, name), name
    h = _native.lib()
    want = int(re.search(r"#define LQ_ABI_VERSION (\d+)", header).group(1))
    assert h.lq_abi_version() == want == _native.ABI_VERSION
    from paper_2404_08867_b200 import engine
    cfg = make_config(5)
    pi = engine.plain_integrand(lq.parse(cfg.text, cfg.d), cfg.d)
    assert _native.lattice_layout(pi.struct, cfg.plain_n)[:3] == (6144, 342, cfg.plain_n)
    prog = engine.plain_integrand(lq.parse(cfg.text, cfg.d), cfg.d, force_program=True)
    assert _native.lattice_layout(prog.struct, cfg.plain_n)[:3] == (4096, 512, cfg.plain_n)


def test_error_mapping_without_gpu():
    from paper_2404_08867_b200 import _native
    if not os.path.exists(_native.LIB_PATH):
        pytest.skip("liblq.so not built")
    import torch
    if torch.cuda.is_available():
        pytest.skip("CPU-only check")
    with pytest.raises(_native.NativeUnavailable):
        _native.ctx(0)


def test_layout_memo_tracks_inputs(monkeypatch):
    # layout_of memoises by input bytes: the same buffers rewritten in place,
    # a different z, and the LQ_FFT / LQ_ORBIT / LQ_PAIR switches must each
    # give a fresh decision, never the remembered one
    import numpy as np
    from paper_2404_08867_b200 import _native, engine
    if not os.path.exists(_native.LIB_PATH):
        pytest.skip("liblq.so not built")
    cfg = make_config(5)
    pi = engine.plain_integrand(lq.parse(cfg.text, cfg.d), cfg.d)
    rule = lq.korobov_vector(cfg.plain_a, cfg.plain_n, cfg.d)
    z = rule.z_reduced_array()
    lay = lambda: _native.lattice_layout(pi.struct, rule.n, z)   # noqa: E731
    assert lay().mode == _native.LAYOUT_ORBIT_FFT
    assert lay().mode == _native.LAYOUT_ORBIT_FFT                 # memo hit
    monkeypatch.setenv("LQ_FFT", "0")
    assert lay().mode == _native.LAYOUT_ORBIT
    monkeypatch.setenv("LQ_ORBIT", "0")
    assert lay().mode == _native.LAYOUT_PAIRED
    monkeypatch.setenv("LQ_PAIR", "0")
    assert lay().mode == _native.LAYOUT_INDEX
    monkeypatch.delenv("LQ_FFT")
    monkeypatch.delenv("LQ_ORBIT")
    monkeypatch.delenv("LQ_PAIR")
    assert lay().mode == _native.LAYOUT_ORBIT_FFT
    beta = pi._keep[0]
    saved = beta.copy()
    try:
        beta *= 1e6                      # fails the FFT accuracy guard: direct orbit kernel
        assert lay().mode == _native.LAYOUT_ORBIT
    finally:
        beta[:] = saved
    assert lay().mode == _native.LAYOUT_ORBIT_FFT
    z2 = z.copy()
    z2[2] = (z2[2] + 1) % rule.n         # no longer a Korobov vector: mirror pairs
    assert _native.lattice_layout(pi.struct, rule.n, z2).mode == _native.LAYOUT_PAIRED
    assert lay().mode == _native.LAYOUT_ORBIT_FFT


def test_layout_selection_without_gpu():
    # host-side layout decisions (no GPU needed): FFT form for cfg5, the
    # accuracy guard keeps huge-coefficient linear forms on the direct orbit
    # kernel, non-Korobov rules get mirror pairs, n = 2^k Korobov rules levels
    import numpy as np
    from paper_2404_08867_b200 import _native, engine
    cfg = make_config(5)
    pi = engine.plain_integrand(lq.parse(cfg.text, cfg.d), cfg.d)
    rule = lq.korobov_vector(cfg.plain_a, cfg.plain_n, cfg.d)
    lay = _native.lattice_layout(pi.struct, rule.n, rule.z_reduced_array())
    assert lay.mode == _native.LAYOUT_ORBIT_FFT and lay.tile_units == 2
    assert lay.n_units * (4097 - cfg.d) >= (rule.n - 1) // 2
    d = 200
    big = "cos(" + " + ".join(f"{30.0 + j}*x[{j + 1}]" for j in range(d)) + ")"
    pib = engine.plain_integrand(lq.parse(big, d), d)
    r = lq.korobov_vector(1234567, 2147483647, d)
    assert _native.lattice_layout(pib.struct, r.n, r.z_reduced_array()).mode == _native.LAYOUT_ORBIT
    r2 = lq.LatticeRule(1000003, tuple(int(v) for v in np.arange(1, 2 * d, 2)))
    assert _native.lattice_layout(pib.struct, r2.n, r2.z_reduced_array()).mode == _native.LAYOUT_PAIRED
    r3 = lq.korobov_vector(7, 1 << 20, d)
    assert _native.lattice_layout(pib.struct, r3.n, r3.z_reduced_array()).mode == _native.LAYOUT_ORBIT_POW2


@pytest.mark.parametrize("fam,n,d,fft", [("expabs", 2147483647, 48, False), ("expabs", 2147483647, 49, True),
                                         ("expabs", 1000003, 111, False), ("expabs", 1000003, 112, True),
                                         ("sincos", 16777213, 56, True), ("sincos", 1000003, 96, False),
                                         ("gauss", 2147483647, 48, False), ("gauss", 2147483647, 64, True),
                                         ("pow", 2147483647, 48, False), ("pow", 2147483647, 49, True),
                                         ("pow", 1000003, 96, False),
                                         ("expabs", 100003, 300, False)])
def test_fft_threshold_without_gpu(fam, n, d, fft):
    # the measured FFT-form crossovers (lq_api.cu fft_min_d, tools/fft_crossover.py)
    from paper_2404_08867_b200 import _native, engine
    c = [0.1 + 0.01 * (j % 7) for j in range(d)]
    if fam == "expabs":
        text = "exp(-abs(" + " + ".join(f"{c[j]!r}*(x[{j + 1}] - 0.5)" for j in range(d)) + "))"
    elif fam == "sincos":
        text = "cos(0.3 + " + " + ".join(f"{c[j]!r}*x[{j + 1}]" for j in range(d)) + ")"
    elif fam == "pow":
        text = "(1.5 + " + " + ".join(f"{c[j] / d!r}*x[{j + 1}]" for j in range(d)) + ")^(-3)"
    else:
        text = "exp(-(" + " + ".join(f"{c[j]!r}*(x[{j + 1}] - 0.5)^2" for j in range(d)) + "))"
    pi = engine.plain_integrand(lq.parse(text, d), d)
    r = lq.korobov_vector(76231, n, d)
    mode = _native.lattice_layout(pi.struct, r.n, r.z_reduced_array()).mode
    assert (mode == _native.LAYOUT_ORBIT_FFT) == fft, mode


def test_fibonacci_rule_mirrors_reference():
    # lattice.py:120-129 and the reference's own pins (tests/test_lattice.py:85-98)
    assert lq.fibonacci_rule(2) == lq.LatticeRule(2, (1, 1))
    assert lq.fibonacci_rule(10) == lq.LatticeRule(89, (1, 55))
    assert lq.fibonacci_rule(15) == lq.LatticeRule(987, (1, 610))
    for k in range(3, 30):
        r = lq.fibonacci_rule(k)
        assert r.z[1] < r.n and math.gcd(r.z[1], r.n) == 1
    with pytest.raises(ValueError):
        lq.fibonacci_rule(1)
    with pytest.raises(OverflowError):
        lq.fibonacci_rule(78)


def test_pow2_layout_without_gpu():
    # n = 2^k Korobov rules get the level layout; even a, composite non-2^k n,
    # or a = +-1 do not
    from paper_2404_08867_b200 import _native, engine
    cfg = make_config(5)
    pi = engine.plain_integrand(lq.parse(cfg.text, cfg.d), cfg.d)
    r = lq.korobov_vector(12345 | 1, 1 << 24, cfg.d)
    lay = _native.lattice_layout(pi.struct, r.n, r.z_reduced_array())
    assert lay.mode == _native.LAYOUT_ORBIT_POW2 and lay.tile_units == 1
    r = lq.korobov_vector(1, 1 << 24, cfg.d)
    assert _native.lattice_layout(pi.struct, r.n, r.z_reduced_array()).mode != _native.LAYOUT_ORBIT_POW2
    r = lq.korobov_vector(12346, 1 << 24, cfg.d)
    assert _native.lattice_layout(pi.struct, r.n, r.z_reduced_array()).mode != _native.LAYOUT_ORBIT_POW2


def test_jit_policy_refuses_long_programs(monkeypatch):
    """NVRTC time grows faster than quadratically with the expression (a
    3000-instruction body took 620 s on the box, the interpreter 3.4 ms):
    past JIT_MAX_INSN the interpreter always runs."""
    from paper_2404_08867_b200 import jit
    monkeypatch.delenv("LQ_JIT", raising=False)
    assert jit.jit_wanted(1e12, 40)
    assert not jit.jit_wanted(1e8, 40)
    assert not jit.jit_wanted(1e15, jit.JIT_MAX_INSN + 1)
    assert not jit.jit_wanted(2e9, 128)            # 16x the base threshold at 128 instructions
    monkeypatch.setenv("LQ_JIT", "always")
    assert jit.jit_wanted(1.0, 10**6)
    monkeypatch.setenv("LQ_JIT", "0")
    assert not jit.jit_wanted(1e15, 10)


# names of latquad.__all__ deliberately not provided: the symbolic algebra and
# the transform validation path (SURVEY §2 / DESIGN §8: never on the value path)
OUT_OF_SCOPE = {"bind", "partial_sum", "substitute", "NonCartesianStructureError", "TransformedIntegrand",
                "build_axis_grids", "forward_transform", "grid_completion", "inverse_substitution",
                "make_transformed_integrand"}


def test_top_level_api_covers_the_reference_exports():
    """A drop-in user's `from latquad import X` works for every value-path name
    the reference exports (/root/reference/pkg/src/latquad/__init__.py)."""
    src = "/root/reference/pkg/src"
    if not os.path.isdir(os.path.join(src, "latquad")):
        pytest.skip("reference not importable here")
    import sys
    sys.path.insert(0, src)
    try:
        import latquad
    finally:
        sys.path.remove(src)
    missing = sorted(set(latquad.__all__) - OUT_OF_SCOPE - set(dir(lq)))
    assert not missing, missing
    assert set(lq.__all__) >= set(latquad.__all__) - OUT_OF_SCOPE
    e = lq.get("invpow")
    assert e.ref(4) == latquad.get("invpow").ref(4) and e.suites == latquad.get("invpow").suites
    assert [x.id for x in lq.entries()] == [x.id for x in latquad.entries()]
    assert lq.eval(lq.parse("exp(1) + 2*pi", 1), {}) == latquad.eval(latquad.parse("exp(1) + 2*pi", 1), {})


def test_reference_import_shim_resolves():
    """tools/refcompat/latquad (the shim that runs the reference's own test
    suite against this package, tools/run_reference_tests.py) imports every
    submodule the reference's tests use, without a GPU."""
    import importlib
    import sys
    shim = os.path.join(REPO, "tools", "refcompat")
    saved = {k: sys.modules.pop(k) for k in [k for k in sys.modules if k == "latquad" or k.startswith("latquad.")]}
    sys.path.insert(0, shim)
    try:
        for name in ("latquad", "latquad.exprcore", "latquad.lattice", "latquad.quad", "latquad.mdi",
                     "latquad.transform", "latquad.corpus", "latquad.bench", "latquad.cli"):
            importlib.import_module(name)
        import latquad
        assert latquad.slr_integrate is lq.slr_integrate
        from latquad.exprcore import make_sum, parse, var
        e = make_sum([(var(1), 2.0), (var(2), 1.0)], 0.5)
        assert e is parse("2*x[1] + x[2] + 0.5", 2)
        assert e.kind == "sum" and e.value == 0.5 and len(e.children) == 2
    finally:
        sys.path.remove(shim)
        for k in [k for k in sys.modules if k == "latquad" or k.startswith("latquad.")]:
            del sys.modules[k]
        sys.modules.update(saved)


def test_composite_modulus_layouts_cover_the_lattice():
    """Korobov rules over composite n: the divisor-class plan (a unit-group
    orbit plan per divisor m of n, plus the small lattice mod m0)
    covers every lattice index exactly once, point and mirror counted
    together (lq_layout_cover, host only) -- for odd, even, prime-power and
    many-factor moduli, direct chains (d = 8) and FFT chains (d = 120)."""
    import ctypes as C
    import math
    import random
    from paper_2404_08867_b200 import _native as N, engine
    if not os.path.exists(N.LIB_PATH):
        pytest.skip("liblq.so not built")
    h = N.lib()
    rng = random.Random(41)
    used = set()
    cases = [(n, 8) for n in (2 * 5**4 * 4, 2 * 3**7, 10000, 4 * 7**5, 12289 * 3, 30030, 65535, 3**10, 5**7,
                              7 * 11 * 13 * 17 * 19, 1000000, 2**20 - 1, 1009 * 1013)]
    cases += [(n, 120) for n in (1000000, 3 * 5 * 7 * 11 * 13 * 17 * 19, 2**22 - 2)]
    for n, d in cases:
        for _ in range(3):
            a = rng.randrange(2, n)
            while math.gcd(a, n) != 1:
                a = rng.randrange(2, n)
            text = "exp(" + " + ".join(f"{0.3 + 0.01 * j}*x[{j + 1}]" for j in range(d)) + ")"
            pi = engine.plain_integrand(lq.parse(text, d), d)
            z = lq.korobov_vector(a, n, d).z_reduced_array()
            miss, rep = C.c_int64(), C.c_int64()
            N.check(h.lq_layout_cover(C.byref(pi.struct), n, N.as_ptr(z), C.byref(miss), C.byref(rep)))
            assert (miss.value, rep.value) == (0, 0), (n, a, d, miss.value, rep.value)
            used.add(N.lattice_layout(pi.struct, n, z).mode)
    assert N.LAYOUT_ORBIT_POW2 in used


def test_jit_source_step_selection():
    # the JIT lattice kernel steps coordinates for expressions of at most
    # STEP_MAX_VARS distinct coordinates: lq_use lists them (0-based, sorted)
    # and lq_fc reads them by rank
    from paper_2404_08867_b200 import jit
    src = jit.source_for(lq.parse("x[7]*exp(x[2]) + x[7]^2", 9))
    assert "#define LQ_STEP 1" in src and "#define LQ_NU 2" in src
    assert "lq_use[LQ_NU] = {1, 6}" in src
    assert "x(0)" in src and "x(1)" in src and "x(6)" in src    # lq_fc by rank, lq_f by index
    wide = jit.source_for(lq.parse("sum(i=1..d, x[i]^2)", jit.STEP_MAX_VARS + 1))
    assert "#define LQ_STEP" not in wide
    assert "#define LQ_STEP" not in jit.source_for(lq.parse("2.5", 3))
