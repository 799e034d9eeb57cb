"""Korobov-orbit kernel (k_orbit) against the oracle and the
per-index kernels.  The orbit kernel sums the same points in a different
order (chains i0 a^k plus their mirrors n - i), so it must agree with the
oracle within the north-star 1e-10 and with the index kernels to rounding."""

import math
import zlib

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

REL = 1e-10


@pytest.fixture(scope="module")
def env():
    import paper_2404_08867_b200 as lq
    from paper_2404_08867_b200 import _native as N, engine
    N.lib()
    return lq, N, engine


def _order(a, n):
    o, m = n - 1, n - 1
    p = 2
    fac = []
    while p * p <= m:
        if m % p == 0:
            fac.append(p)
            while m % p == 0:
                m //= p
        p += 1
    if m > 1:
        fac.append(m)
    for p in fac:
        while o % p == 0 and pow(a, o // p, n) == 1:
            o //= p
    return o


def _sum(lq, engine, f, rule, mode, monkeypatch):
    monkeypatch.setenv("LQ_ORBIT", mode)
    pi = engine.plain_integrand(f, rule.d)
    return engine.lattice_sum(pi, rule.n, rule.z_reduced_array())


def _layout(N, engine, f, rule):
    pi = engine.plain_integrand(f, rule.d)
    return N.lattice_layout(pi.struct, rule.n, rule.z_reduced_array())


@pytest.mark.parametrize("cid", [1, 2, 3])
def test_orbit_configs_vs_oracle(env, cid, monkeypatch):
    lq, N, engine = env
    from paper_2404_08867_b200.configs import make_config
    from oracle import np_oracle
    cfg = make_config(cid)
    f = lq.parse(cfg.text, cfg.d)
    rule = lq.korobov_vector(cfg.plain_a, cfg.plain_n, cfg.d)
    monkeypatch.setenv("LQ_ORBIT", "always")
    assert _layout(N, engine, f, rule).mode == N.LAYOUT_ORBIT
    orb = _sum(lq, engine, f, rule, "always", monkeypatch)
    idx = _sum(lq, engine, f, rule, "0", monkeypatch)
    assert math.isclose(orb, idx, rel_tol=1e-12), (orb, idx)
    if cfg.plain_n <= 20000:
        ref = np_oracle.slr_sum(f, rule.n, list(rule.z_reduced))
        assert math.isclose(orb, ref, rel_tol=REL), (orb, ref)


@pytest.mark.parametrize("kind", ["primitive", "odd_order", "even_order_cosets"])
@pytest.mark.parametrize("family", ["exp", "sincos", "expabs", "gauss"])
def test_orbit_group_structures(env, kind, family, monkeypatch):
    # prime n = 100003, n - 1 = 2 * 3 * 7 * 2381; a chosen for each coset structure
    lq, N, engine = env
    from oracle import np_oracle
    n, d = 100003, 37
    g = 2
    while any(pow(g, (n - 1) // p, n) == 1 for p in (2, 3, 7, 2381)):
        g += 1
    a = {"primitive": g, "odd_order": pow(g, 2, n), "even_order_cosets": pow(g, 3, n)}[kind]
    o = _order(a, n)
    assert (o == n - 1) if kind == "primitive" else (o % 2 == (1 if kind == "odd_order" else 0))
    rng = np.random.default_rng(zlib.crc32(f"{kind}/{family}".encode()))
    c = [float(v) for v in rng.uniform(0, 1, d)]
    w = [float(v) for v in rng.uniform(0, 1, d)]
    if family == "exp":
        text = "exp(" + " + ".join(f"{c[j] / d!r}*x[{j + 1}]" for j in range(d)) + ")"
    elif family == "sincos":
        text = "cos(0.7 + " + " + ".join(f"{c[j]!r}*x[{j + 1}]" for j in range(d)) + ")"
    elif family == "expabs":
        text = "exp(-abs(" + " + ".join(f"{c[j] / 4!r}*(x[{j + 1}] - {w[j]!r})" for j in range(d)) + "))"
    else:
        text = "exp(-(" + " + ".join(f"{c[j] ** 2 / 4!r}*(x[{j + 1}] - {w[j]!r})^2" for j in range(d)) + "))"
    f = lq.parse(text, d)
    rule = lq.korobov_vector(a, n, d)
    monkeypatch.setenv("LQ_ORBIT", "always")
    lay = _layout(N, engine, f, rule)
    assert lay.mode == N.LAYOUT_ORBIT, (kind, o)
    orb = _sum(lq, engine, f, rule, "always", monkeypatch)
    idx = _sum(lq, engine, f, rule, "0", monkeypatch)
    ref = np_oracle.slr_sum(f, rule.n, list(rule.z_reduced))
    assert math.isclose(orb, ref, rel_tol=REL), (kind, family, orb, ref)
    assert math.isclose(orb, idx, rel_tol=1e-12), (kind, family, orb, idx)


def test_orbit_not_used_for_non_korobov_or_composite(env, monkeypatch):
    lq, N, engine = env
    monkeypatch.setenv("LQ_ORBIT", "always")
    f = lq.parse("exp(0.1*x[1] + 0.2*x[2] + 0.3*x[3])", 3)
    # composite n
    r = lq.korobov_vector(5, 100000, 3)
    assert _layout(N, engine, f, r).mode == N.LAYOUT_INDEX
    # not a Korobov vector
    r = lq.LatticeRule(100003, (1, 17, 1234))
    assert _layout(N, engine, f, r).mode == N.LAYOUT_INDEX
    # a = 1: every point its own coset (too many cosets) -> index kernels
    r = lq.korobov_vector(1, 100003, 3)
    assert _layout(N, engine, f, r).mode == N.LAYOUT_INDEX
    # sub-ranges never use the orbit kernel, full ranges do
    r = lq.korobov_vector(7, 100003, 3)
    pi = engine.plain_integrand(f, 3)
    z = r.z_reduced_array()
    half = engine.lattice_sum(pi, r.n, z, 0, 50000) + engine.lattice_sum(pi, r.n, z, 50000, r.n)
    full = engine.lattice_sum(pi, r.n, z)
    assert math.isclose(half, full, rel_tol=1e-13)


def test_orbit_cfg5_matches_index_kernel(env, monkeypatch):
    # the headline lattice: 2^31 - 1 points, d = 1000
    lq, N, engine = env
    from paper_2404_08867_b200.configs import make_config
    cfg = make_config(5)
    f = lq.parse(cfg.text, cfg.d)
    rule = lq.korobov_vector(cfg.plain_a, cfg.plain_n, cfg.d)
    monkeypatch.delenv("LQ_ORBIT", raising=False)
    assert _layout(N, engine, f, rule).mode == N.LAYOUT_ORBIT
    orb = _sum(lq, engine, f, rule, "1", monkeypatch)
    idx = _sum(lq, engine, f, rule, "0", monkeypatch)
    assert math.isclose(orb, idx, rel_tol=1e-12), (orb, idx)
