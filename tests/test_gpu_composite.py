"""GPU: Korobov rules over composite n through the divisor-class plan
(a unit-group orbit level per divisor of n, direct or FFT-form
chains, plus the small lattice mod m0) against the mirror-paired index kernel
(LQ_ORBIT=0) at 1e-12 and the oracle / the reference's own sums at 1e-10."""

import math
import random

import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lq():
    import paper_2404_08867_b200 as m
    return m


def _text(family, d, rng):
    c = [rng.uniform(0.2, 1.0) * 3.0 / d for _ in range(d)]
    lin = " + ".join(f"{cj!r}*x[{j + 1}]" for j, cj in enumerate(c))
    if family == "exp":
        return f"exp(-0.5 + {lin})"
    if family == "expabs":
        return f"exp(-abs({lin} - 1.2))"
    if family == "cos":
        return f"cos(0.3 + {lin})"
    q = " + ".join(f"{-rng.uniform(0.0, 1.0) * 3.0 / d!r}*x[{j + 1}]^2" for j in range(d))
    return f"exp({lin} + {q})"


def _sums(lq, text, d, n, a, monkeypatch):
    from paper_2404_08867_b200 import _native as N, engine
    f = lq.parse(text, d)
    rule = lq.korobov_vector(a, n, d)
    z = rule.z_reduced_array()
    pi = engine.plain_integrand(f, d)
    mode = N.lattice_layout(pi.struct, n, z).mode
    got = engine.lattice_sum(pi, n, z)
    monkeypatch.setenv("LQ_ORBIT", "0")
    ref = engine.lattice_sum(engine.plain_integrand(f, d), n, z)
    monkeypatch.delenv("LQ_ORBIT")
    return mode, got, ref


@pytest.mark.parametrize("n,d", [(10000, 8), (1000000, 20), (2 * 3**7 * 11, 12), (3 * 5 * 7 * 11 * 13 * 17 * 19, 16),
                                 (2**22 - 2, 120), (1000000, 150), (6 * 7**7, 64)])
@pytest.mark.parametrize("family", ["exp", "expabs", "cos", "quad"])
def test_composite_modulus_matches_paired_kernel(lq, n, d, family, monkeypatch):
    from paper_2404_08867_b200 import _native as N
    rng = random.Random(n * 7 + d)
    a = rng.randrange(2, n)
    while math.gcd(a, n) != 1:
        a = rng.randrange(2, n)
    mode, got, ref = _sums(lq, _text(family, d, rng), d, n, a, monkeypatch)
    assert mode == N.LAYOUT_ORBIT_POW2, (n, a, d, mode)
    assert math.isclose(got, ref, rel_tol=1e-12, abs_tol=1e-12 * n), (n, d, family, got, ref)


def test_composite_modulus_against_the_oracle(lq, monkeypatch):
    from oracle import np_oracle as orc
    rng = random.Random(5)
    for n, d in [(10000, 8), (30030, 6), (2 * 3**7 * 11, 10)]:
        a = rng.randrange(2, n)
        while math.gcd(a, n) != 1:
            a = rng.randrange(2, n)
        text = _text("expabs", d, rng)
        got = lq.slr_integrate(lq.parse(text, d), lq.korobov_vector(a, n, d)).value
        want = orc.slr_value(text, n, [a**j for j in range(d)])
        assert abs(got - want) <= 1e-10 * abs(want), (n, d, got, want)


def test_composite_cfg5_scale(lq, monkeypatch):
    """Config 5's integrand over n = 2^31 - 2 (= 2 3^2 7 11 31 151 331): the
    FFT-form chains of every divisor class against the paired kernel."""
    from paper_2404_08867_b200 import _native as N
    from paper_2404_08867_b200.configs import make_config
    cfg = make_config(5)
    n = 2**31 - 2
    rng = random.Random(9)
    a = rng.randrange(2, n)
    while math.gcd(a, n) != 1:
        a = rng.randrange(2, n)
    mode, got, ref = _sums(lq, cfg.text, cfg.d, n, a, monkeypatch)
    assert mode == N.LAYOUT_ORBIT_POW2
    assert math.isclose(got, ref, rel_tol=1e-12), (got, ref)


@pytest.mark.parametrize("n,d", [(10**8, 1000), (3 * 5 * 7 * 11 * 13 * 17 * 19 * 4, 40)])
def test_composite_partials_sharded_bit_identical(lq, n, d, monkeypatch):
    """The divisor-class layout through the multi-GPU building blocks: three
    shards of its super-chunks (levels with FFT-form and direct chains, the
    small lattice) reproduce the one-launch sum bit for bit."""
    import ctypes as C
    import torch
    from paper_2404_08867_b200 import _native as N, engine
    from paper_2404_08867_b200.distributed import shard_range
    rng = random.Random(n)
    a = rng.randrange(2, n)
    while math.gcd(a, n) != 1:
        a = rng.randrange(2, n)
    f = lq.parse(_text("expabs", d, rng), d)
    z = lq.korobov_vector(a, n, d).z_reduced_array()
    pi = engine.plain_integrand(f, d)
    lay = N.lattice_layout(pi.struct, n, z)
    assert lay.mode == N.LAYOUT_ORBIT_POW2 and lay.n_supers >= 2, lay
    h, ctx = N.lib(), N.ctx()
    S = lay.n_supers
    one = torch.zeros(S, dtype=torch.float64, device="cuda")
    N.check(h.lq_lattice_partials(ctx, C.byref(pi.struct), n, N.as_ptr(z), 0, S, C.c_void_p(one.data_ptr())))
    many = torch.zeros(S, dtype=torch.float64, device="cuda")
    for r in range(3):
        lo, hi = shard_range(S, r, 3)
        N.check(h.lq_lattice_partials(ctx, C.byref(pi.struct), n, N.as_ptr(z), lo, hi,
                                      C.c_void_p(many.data_ptr() + 8 * lo)))
    torch.cuda.synchronize()
    assert torch.equal(one.view(torch.int64), many.view(torch.int64))
    out = C.c_double()
    N.check(h.lq_reduce_sum(ctx, C.c_void_p(one.data_ptr()), S, C.byref(out)))
    assert out.value == engine.lattice_sum(pi, n, z)


def test_composite_modulus_program_outer(lq, monkeypatch):
    """A function of one linear form outside the closed families (the outer G
    as bytecode, FFT-form chains only) over a composite modulus: the classes
    with long orbits take FFT chains, the rest the small lattice."""
    from paper_2404_08867_b200 import _native as N
    rng = random.Random(77)
    n, d = 10**8, 200
    a = rng.randrange(2, n)
    while math.gcd(a, n) != 1:
        a = rng.randrange(2, n)
    c = [rng.uniform(0.2, 1.0) * 3.0 / d for _ in range(d)]
    lin = " + ".join(f"{cj!r}*x[{j + 1}]" for j, cj in enumerate(c))
    mode, got, ref = _sums(lq, f"1/(1 + (2*({lin}) - 0.8)^2)", d, n, a, monkeypatch)
    assert mode == N.LAYOUT_ORBIT_POW2, mode
    assert math.isclose(got, ref, rel_tol=1e-12), (got, ref)
