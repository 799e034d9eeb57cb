"""FFT form of the Korobov chain sums (k_orbit_fft) against
the direct orbit kernel and the oracle.  The correlation through an FFT is
exact up to rounding (~1e-14 relative on the linear forms), so sums agree with
the direct kernels to 1e-12 and with the oracle to the north-star 1e-10."""

import math
import zlib

import numpy as np
import pytest

from test_gpu_orbit import _family_text, _order

pytestmark = pytest.mark.gpu

REL = 1e-10


@pytest.fixture(scope="module")
def env():
    import paper_2404_08867_b200 as lq
    from paper_2404_08867_b200 import _native as N, engine
    N.lib()
    return lq, N, engine


def _sums(engine, N, pi, n, z, monkeypatch):
    out = {}
    for fft in ("always", "0"):
        monkeypatch.setenv("LQ_FFT", fft)
        out[N.lattice_layout(pi.struct, n, z).mode] = engine.lattice_sum(pi, n, z)
    return out


@pytest.mark.parametrize("family", ["exp", "sincos", "expabs", "pow", "gauss", "qtrig"])
@pytest.mark.parametrize("n,d,kind", [(100003, 37, "primitive"), (100003, 200, "odd_order"),
                                      (1000003, 600, "even_order_cosets"), (1000003, 2048, "primitive")])
def test_fft_matches_direct_orbit_and_oracle(env, family, n, d, kind, monkeypatch):
    lq, N, engine = env
    from oracle import np_oracle
    fac = {100003: (2, 3, 7, 2381), 1000003: (2, 3, 166667)}[n]
    g = 2
    while any(pow(g, (n - 1) // p, n) == 1 for p in fac):
        g += 1
    a = {"primitive": g, "odd_order": pow(g, 2, n), "even_order_cosets": pow(g, 3, n)}[kind]
    rng = np.random.default_rng(zlib.crc32(f"{family}/{n}/{d}".encode()))
    f = lq.parse(_family_text(family, d, rng), d)
    rule = lq.korobov_vector(a, n, d)
    pi = engine.plain_integrand(f, d)
    z = rule.z_reduced_array()
    got = _sums(engine, N, pi, n, z, monkeypatch)
    # without the FFT form: the direct orbit kernel, or mirror pairs where its
    # parameter-space tables cannot hold d (Gaussian family, d = 2048)
    assert N.LAYOUT_ORBIT_FFT in got and len(got) == 2, got.keys()
    fft = got.pop(N.LAYOUT_ORBIT_FFT)
    (direct,) = got.values()
    assert math.isclose(fft, direct, rel_tol=1e-12, abs_tol=1e-12 * n), (family, n, d, fft, direct)
    if n * d <= 3_000_000:
        ref = np_oracle.slr_sum(f, n, list(rule.z_reduced))
        assert math.isclose(fft, ref, rel_tol=REL, abs_tol=1e-10 * n), (family, n, d, fft, ref)


def test_fft_cfg5(env, monkeypatch):
    # the headline lattice through the FFT form vs the direct orbit kernel
    lq, N, engine = env
    from paper_2404_08867_b200.configs import make_config
    cfg = make_config(5)
    f = lq.parse(cfg.text, cfg.d)
    rule = lq.korobov_vector(cfg.plain_a, cfg.plain_n, cfg.d)
    pi = engine.plain_integrand(f, cfg.d)
    got = _sums(engine, N, pi, rule.n, rule.z_reduced_array(), monkeypatch)
    fft, direct = got[N.LAYOUT_ORBIT_FFT], got[N.LAYOUT_ORBIT]
    assert math.isclose(fft, direct, rel_tol=1e-12), (fft, direct)


def test_fft_gaussian_large(env, monkeypatch):
    # config 3's integrand on a 2^27-point Korobov lattice: FFT form vs direct orbit
    lq, N, engine = env
    from paper_2404_08867_b200.configs import make_config
    cfg = make_config(3)
    f = lq.parse(cfg.text, cfg.d)
    n = 134217689
    rule = lq.korobov_vector(cfg.plain_a % n, n, cfg.d)
    pi = engine.plain_integrand(f, cfg.d)
    got = _sums(engine, N, pi, n, rule.z_reduced_array(), monkeypatch)
    fft, direct = got[N.LAYOUT_ORBIT_FFT], got[N.LAYOUT_ORBIT]
    assert math.isclose(fft, direct, rel_tol=1e-12), (fft, direct)


def _pair_text(family, d, rng, scale, offset):
    c = rng.uniform(0, 1, d)
    c = c * (scale / c.sum())
    w = rng.uniform(0, 1, d)
    if family == "expabs":
        return "exp(-abs(" + " + ".join(f"{float(c[j])!r}*(x[{j + 1}] - {float(w[j])!r})" for j in range(d)) + "))"
    sgn = np.where(rng.uniform(size=d) < 0.5, -1.0, 1.0)
    if family == "exp":
        return f"exp({offset!r} + " + " + ".join(f"{float(sgn[j] * c[j])!r}*x[{j + 1}]" for j in range(d)) + ")"
    return "2.0 + 0.5*cos(1.3 + " + " + ".join(f"{float(sgn[j] * c[j])!r}*x[{j + 1}]" for j in range(d)) + ")"


@pytest.mark.parametrize("family,scale,offset", [("expabs", 10.0, 0), ("expabs", 0.01, 0), ("expabs", 350.0, 0),
                                                 ("expabs", 800.0, 0), ("exp", 3.0, 0.25), ("exp", 600.0, 0.25),
                                                 ("exp", 100.0, -650.0), ("sincos", 9.0, 0), ("sincos", 400.0, 0)])
def test_fft_pair_fast(env, family, scale, offset, monkeypatch):
    # the one-reduction point/mirror outer (PairFast) against
    # the two-exp form and the oracle; bounds past the normal range (|y| <= 700:
    # expabs 800, exp offset -650) fall back to the two-exp form
    lq, N, engine = env
    from oracle import np_oracle
    n, d, a = 100003, 150, 2
    rng = np.random.default_rng(zlib.crc32(f"pair/{family}/{scale}".encode()))
    f = lq.parse(_pair_text(family, d, rng, scale, offset), d)
    rule = lq.korobov_vector(a, n, d)
    pi = engine.plain_integrand(f, d)
    z = rule.z_reduced_array()
    monkeypatch.setenv("LQ_FFT", "always")
    assert N.lattice_layout(pi.struct, n, z).mode == N.LAYOUT_ORBIT_FFT
    fast = engine.lattice_sum(pi, n, z)
    monkeypatch.setenv("LQ_PAIRFAST", "0")
    slow = engine.lattice_sum(pi, n, z)
    assert math.isclose(fast, slow, rel_tol=1e-13, abs_tol=1e-300), (fast, slow)
    ref = np_oracle.slr_sum(f, n, list(rule.z_reduced))
    assert math.isclose(fast, ref, rel_tol=REL, abs_tol=1e-300), (fast, ref)


@pytest.mark.parametrize("family", ["exp", "expabs", "sincos"])
@pytest.mark.parametrize("d", [768, 769, 1024, 1025])
def test_fft_position_bound_boundaries(env, family, d, monkeypatch):
    """The compile-time bound RM on the positions a chain reaches (RM * 256 >=
    B = 4097 - d; RM = 16 / 13 / 13 / 12 at these d) drops the dead outputs of
    the last inverse pass: the sums must not change at the switch points."""
    lq, N, engine = env
    n, g = 100003, 2
    while any(pow(g, (n - 1) // p, n) == 1 for p in (2, 3, 7, 2381)):
        g += 1
    rng = np.random.default_rng(zlib.crc32(f"rm/{family}/{d}".encode()))
    f = lq.parse(_family_text(family, d, rng), d)
    rule = lq.korobov_vector(g, n, d)
    pi = engine.plain_integrand(f, d)
    got = _sums(engine, N, pi, n, rule.z_reduced_array(), monkeypatch)
    fft = got.pop(N.LAYOUT_ORBIT_FFT)
    (direct,) = got.values()
    assert math.isclose(fft, direct, rel_tol=1e-12, abs_tol=1e-12 * n), (family, d, fft, direct)
