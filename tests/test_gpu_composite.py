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
