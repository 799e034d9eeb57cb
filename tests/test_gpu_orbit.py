"""Korobov-orbit kernel (k_orbit) against the oracle and the
per-index kernels.  The orbit kernel sums the same points in a different
order (chains i0 a^k plus their mirrors n - i), so it must agree with the
oracle within the north-star 1e-10 and with the index kernels to rounding."""

import math
import zlib

import numpy as np
import pytest

import fft_cases

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
    monkeypatch.setenv("LQ_FFT", "0")          # the direct orbit kernel (the FFT form: test_gpu_fft.py)
    assert _layout(N, engine, f, rule).mode == N.LAYOUT_ORBIT
    orb = _sum(lq, engine, f, rule, "always", monkeypatch)
    idx = _sum(lq, engine, f, rule, "0", monkeypatch)
    assert math.isclose(orb, idx, rel_tol=1e-12), (orb, idx)
    if cfg.plain_n <= 20000:
        ref = np_oracle.slr_sum(cfg.text, rule.n, list(rule.z_reduced))
        assert math.isclose(orb, ref, rel_tol=REL), (orb, ref)


@pytest.mark.parametrize("kind", ["primitive", "odd_order", "even_order_cosets"])
@pytest.mark.parametrize("family", ["exp", "sincos", "expabs", "gauss", "pow", "qtrig"])
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
    text = _family_text(family, d, rng)
    f = lq.parse(text, d)
    rule = lq.korobov_vector(a, n, d)
    monkeypatch.setenv("LQ_ORBIT", "always")
    lay = _layout(N, engine, f, rule)
    assert lay.mode == N.LAYOUT_ORBIT, (kind, o)
    orb = _sum(lq, engine, f, rule, "always", monkeypatch)
    idx = _sum(lq, engine, f, rule, "0", monkeypatch)
    ref = np_oracle.slr_sum(text, rule.n, list(rule.z_reduced))
    assert math.isclose(orb, ref, rel_tol=REL), (kind, family, orb, ref)
    assert math.isclose(orb, idx, rel_tol=1e-12), (kind, family, orb, idx)


def test_orbit_not_used_for_non_korobov_or_composite(env, monkeypatch):
    lq, N, engine = env
    monkeypatch.setenv("LQ_ORBIT", "always")
    f = lq.parse("exp(0.1*x[1] + 0.2*x[2] + 0.3*x[3])", 3)
    # composite n (and z_j = 5^j shares factors with n: no mirror pairs either)
    r = lq.korobov_vector(5, 100000, 3)
    assert _layout(N, engine, f, r).mode == N.LAYOUT_INDEX
    # not a Korobov vector: mirror pairs only
    r = lq.LatticeRule(100003, (1, 17, 1234))
    assert _layout(N, engine, f, r).mode == N.LAYOUT_PAIRED
    # a = 1: every point its own coset (too many cosets) -> mirror pairs only
    r = lq.korobov_vector(1, 100003, 3)
    assert _layout(N, engine, f, r).mode == N.LAYOUT_PAIRED
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
    monkeypatch.setenv("LQ_FFT", "0")          # the direct orbit kernel (the FFT form: test_gpu_fft.py)
    assert _layout(N, engine, f, rule).mode == N.LAYOUT_ORBIT
    orb = _sum(lq, engine, f, rule, "1", monkeypatch)
    idx = _sum(lq, engine, f, rule, "0", monkeypatch)
    assert math.isclose(orb, idx, rel_tol=1e-12), (orb, idx)


# ---------------------------------------------------------------- mirror pairs
# Rules that are not Korobov-over-a-prime (CBC-built vectors, composite or
# power-of-two n) still pair each point with its mirror when every z_j is a
# unit mod n (LAYOUT_PAIRED, k_fam<PAIR>).

def _family_text(family, d, rng):
    return fft_cases.family_text(family, d, rng)[0]


def _pair_text(family, d, rng, scale, offset):
    return fft_cases.pair_text(family, d, rng, scale, offset)[0]


def _unit_vector(n, d, rng):
    z = [1]
    while len(z) < d:
        v = int(rng.integers(1, n))
        if math.gcd(v, n) == 1:
            z.append(v)
    return tuple(z)


@pytest.mark.parametrize("n", [65536, 100003, 99991 * 2, 3 ** 10])
@pytest.mark.parametrize("family", ["exp", "sincos", "expabs", "gauss", "pow", "qtrig"])
def test_paired_layout_vs_oracle(env, n, family, monkeypatch):
    lq, N, engine = env
    from oracle import np_oracle
    d = 96 if family in ("gauss", "qtrig") else 40       # 96: the cluster split runs too
    rng = np.random.default_rng(zlib.crc32(f"{n}/{family}".encode()))
    text = _family_text(family, d, rng)
    f = lq.parse(text, d)
    rule = lq.LatticeRule(n, _unit_vector(n, d, rng))
    monkeypatch.delenv("LQ_PAIR", raising=False)
    assert _layout(N, engine, f, rule).mode == N.LAYOUT_PAIRED
    pi = engine.plain_integrand(f, d)
    z = rule.z_reduced_array()
    paired = engine.lattice_sum(pi, n, z)
    monkeypatch.setenv("LQ_PAIR", "0")
    assert _layout(N, engine, f, rule).mode == N.LAYOUT_INDEX
    plain = engine.lattice_sum(pi, n, z)
    ref = np_oracle.slr_sum(text, n, list(rule.z_reduced))
    assert math.isclose(paired, ref, rel_tol=REL), (n, family, paired, ref)
    assert math.isclose(paired, plain, rel_tol=1e-12), (n, family, paired, plain)


def test_paired_needs_units(env, monkeypatch):
    lq, N, engine = env
    monkeypatch.delenv("LQ_PAIR", raising=False)
    f = lq.parse("exp(0.1*x[1] + 0.2*x[2])", 2)
    assert _layout(N, engine, f, lq.LatticeRule(1000, (1, 3))).mode == N.LAYOUT_PAIRED
    assert _layout(N, engine, f, lq.LatticeRule(1000, (1, 4))).mode == N.LAYOUT_INDEX   # gcd(4, 1000) > 1
    # a bytecode integrand never pairs
    g = lq.parse("x[1]*x[2] + 1", 2)
    assert _layout(N, engine, g, lq.LatticeRule(1000, (1, 3))).mode == N.LAYOUT_INDEX


def test_paired_partials_sharded_bit_identical(env, monkeypatch):
    import ctypes as C
    import torch
    lq, N, engine = env
    from paper_2404_08867_b200.distributed import shard_range
    monkeypatch.delenv("LQ_PAIR", raising=False)
    n, d = 1 << 26, 64
    rng = np.random.default_rng(11)
    text = _family_text("expabs", d, rng)
    f = lq.parse(text, d)
    rule = lq.LatticeRule(n, _unit_vector(n, d, rng))
    pi = engine.plain_integrand(f, d)
    z = rule.z_reduced_array()
    lay = N.lattice_layout(pi.struct, n, z)
    assert lay.mode == N.LAYOUT_PAIRED and lay.n_units == n // 2 + 1 and lay.n_supers > 4
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
    full = engine.lattice_sum(pi, n, z)
    assert out.value == full
    monkeypatch.setenv("LQ_PAIR", "0")
    assert math.isclose(engine.lattice_sum(pi, n, z), full, rel_tol=1e-12)


@pytest.mark.parametrize("family,kind", [("pow", "lin_pow"), ("qtrig", "quad_sincos")])
def test_new_families_match_bytecode(env, family, kind, monkeypatch):
    # the family kernels against the bytecode interpreter on a sub-range (index
    # layout) and on the full lattice (orbit layout)
    lq, N, engine = env
    d, n = 50, 1000003
    rng = np.random.default_rng(9)
    text = _family_text(family, d, rng)
    f = lq.parse(text, d)
    rule = lq.korobov_vector(76543, n, d)
    fam = engine.plain_integrand(f, d)
    prog = engine.plain_integrand(f, d, force_program=True)
    assert fam.kind == kind
    z = rule.z_reduced_array()
    monkeypatch.setenv("LQ_JIT", "0")
    for lo, hi in ((0, n), (12345, 400000)):
        a = engine.lattice_sum(fam, n, z, lo, hi)
        b = engine.lattice_sum(prog, n, z, lo, hi)
        assert math.isclose(a, b, rel_tol=1e-12), (family, lo, hi, a, b)


@pytest.mark.parametrize("n,d,a", [(5, 3, 2), (7, 1, 3), (2, 4, 1), (3, 2, 2), (4, 3, 3), (1009, 4100, 478),
                                   (100003, 4100, 7)])
def test_layout_edges_vs_index_kernel(env, n, d, a, monkeypatch):
    # tiny moduli (self-mirrored points, no orbit), d = 1, and d beyond the
    # parameter-space tables (global-memory tables): every layout liblq picks
    # equals the plain per-index sum
    lq, N, engine = env
    rng = np.random.default_rng(n + d)
    text = _family_text("expabs", d, rng)
    f = lq.parse(text, d)
    rule = lq.korobov_vector(a, n, d)
    pi = engine.plain_integrand(f, d)
    z = rule.z_reduced_array()
    monkeypatch.delenv("LQ_PAIR", raising=False)
    monkeypatch.delenv("LQ_ORBIT", raising=False)
    lay = N.lattice_layout(pi.struct, n, z)
    got = engine.lattice_sum(pi, n, z)
    monkeypatch.setenv("LQ_PAIR", "0")
    monkeypatch.setenv("LQ_ORBIT", "0")
    assert N.lattice_layout(pi.struct, n, z).mode == N.LAYOUT_INDEX
    want = engine.lattice_sum(pi, n, z)
    assert math.isclose(got, want, rel_tol=1e-12), (n, d, lay, got, want)
    if n * d <= 200000:
        from oracle import np_oracle
        ref = np_oracle.slr_sum(text, n, list(rule.z_reduced))
        assert math.isclose(got, ref, rel_tol=REL), (n, d, got, ref)


@pytest.mark.parametrize("text,d", [
    ("prod(i=1..d, 1/(0.81 + (x[i]-0.6)^2))", 10),                                   # corpus ratprod
    ("(0.81 + x[1]^2 - 1.2*x[1])^(-2) * (2 + x[2]^2)^(-2) * 3", 2),
    ("prod(i=1..d, (0.3 + (x[i]-0.25)^2))", 40),
    ("prod(i=1..d, 1/(0.0001 + (x[i]-0.5)^2))", 6),                                  # sharp peaks
])
def test_product_family_vs_bytecode_and_oracle(env, text, d, monkeypatch):
    lq, N, engine = env
    from oracle import np_oracle
    f = lq.parse(text, d)
    fam = engine.plain_integrand(f, d)
    assert fam.kind == "prod_quad"
    prog = engine.plain_integrand(f, d, force_program=True)
    monkeypatch.setenv("LQ_JIT", "0")
    for n, a in ((10007, 1234), (1000003, 76543)):
        rule = lq.korobov_vector(a, n, d)
        z = rule.z_reduced_array()
        got = engine.lattice_sum(fam, n, z)
        want = engine.lattice_sum(prog, n, z)
        assert math.isclose(got, want, rel_tol=1e-12), (text, n, got, want)
        if n * d <= 200000:
            ref = np_oracle.slr_sum(text, n, list(rule.z_reduced))
            assert math.isclose(got, ref, rel_tol=REL), (text, n, got, ref)


def test_product_family_config4_integrand(env, monkeypatch):
    # config 4's product peak: factors ~ 10^2..10^5, so the running product needs
    # the exponent renormalisation.  All 500 factors underflow the sum to 0.0 in
    # FP64 (reference-identical): the first 90 factors keep
    # it representable (~1e-248).
    lq, N, engine = env
    from paper_2404_08867_b200.configs import make_config
    cfg = make_config(4)
    d = 90
    text = " * ".join(cfg.text.split(" * ")[:d])
    f = lq.parse(text, d)
    fam = engine.plain_integrand(f, d)
    assert fam.kind == "prod_quad"
    prog = engine.plain_integrand(f, d, force_program=True)
    monkeypatch.setenv("LQ_JIT", "0")
    for n, a in ((100003, 3), (1 << 20, 5)):
        rule = lq.korobov_vector(a, n, d)
        z = rule.z_reduced_array()
        got = engine.lattice_sum(fam, rule.n, z)
        want = engine.lattice_sum(prog, rule.n, z)
        assert got > 0.0 and math.isclose(got, want, rel_tol=1e-11), (n, got, want)


def test_randomised_layouts_agree(env, monkeypatch):
    # random primes, Korobov parameters, dimensions and families: the FFT-form
    # orbit, direct orbit, mirror-paired and plain index layouts give the same sums
    lq, N, engine = env
    rng = np.random.default_rng(2024)

    def is_prime(m):
        if m < 2:
            return False
        p = 2
        while p * p <= m:
            if m % p == 0:
                return False
            p += 1
        return True

    fams = ["exp", "sincos", "expabs", "gauss", "pow", "qtrig"]
    for trial in range(24):
        n = int(rng.integers(20000, 2000000))
        while not is_prime(n):
            n += 1
        a = int(rng.integers(2, n - 1))
        d = int(rng.integers(2, 160))
        fam = fams[trial % len(fams)]
        f = lq.parse(_family_text(fam, d, rng), d)
        rule = lq.korobov_vector(a, n, d)
        pi = engine.plain_integrand(f, d)
        z = rule.z_reduced_array()
        vals = {}
        for orb, pair, fft in (("1", "1", "always"), ("1", "1", "0"), ("0", "1", "0"), ("0", "0", "0")):
            monkeypatch.setenv("LQ_ORBIT", orb)
            monkeypatch.setenv("LQ_PAIR", pair)
            monkeypatch.setenv("LQ_FFT", fft)
            mode = N.lattice_layout(pi.struct, n, z).mode
            vals[mode] = engine.lattice_sum(pi, n, z)
        base = vals[N.LAYOUT_INDEX]
        for mode, v in vals.items():
            assert math.isclose(v, base, rel_tol=1e-11, abs_tol=1e-9 * n), (trial, fam, n, a, d, mode, v, base)


# ---------------------------------------------------------------- n = 2^k
@pytest.mark.parametrize("k,a,d", [(12, 5, 9), (16, 3, 37), (20, 1234567 | 1, 37), (20, 3, 200), (22, 5, 300),
                                   (24, 12345 | 1, 600)])
@pytest.mark.parametrize("family", ["exp", "sincos", "expabs", "pow", "gauss", "qtrig"])
def test_pow2_levels_vs_paired(env, k, a, d, family, monkeypatch):
    # Korobov rules with n = 2^k: orbit / FFT levels of the unit groups mod 2^m
    # plus the small 2^m0 lattice against the mirror-paired index kernel
    lq, N, engine = env
    n = 1 << k
    rng = np.random.default_rng(zlib.crc32(f"pow2/{k}/{a}/{d}/{family}".encode()))
    text = _family_text(family, d, rng)
    f = lq.parse(text, d)
    rule = lq.korobov_vector(a % n, n, d)
    pi = engine.plain_integrand(f, d)
    z = rule.z_reduced_array()
    monkeypatch.delenv("LQ_ORBIT", raising=False)
    monkeypatch.delenv("LQ_FFT", raising=False)
    lay = N.lattice_layout(pi.struct, n, z)
    got = engine.lattice_sum(pi, n, z)
    monkeypatch.setenv("LQ_ORBIT", "0")
    assert N.lattice_layout(pi.struct, n, z).mode == N.LAYOUT_PAIRED
    want = engine.lattice_sum(pi, n, z)
    assert lay.mode == N.LAYOUT_ORBIT_POW2, lay
    assert math.isclose(got, want, rel_tol=1e-11, abs_tol=1e-9 * n), (k, a, d, family, got, want)
    if n * d <= 200000:
        from oracle import np_oracle
        ref = np_oracle.slr_sum(text, n, list(rule.z_reduced))
        assert math.isclose(got, ref, rel_tol=REL, abs_tol=1e-9 * n), (k, a, d, family, got, ref)


def test_pow2_partials_sharded_bit_identical(env, monkeypatch):
    # the 2^k layout through the multi-GPU building blocks: shards of tiles
    # (levels and the small lattice) reproduce the one-launch sum bit for bit
    import ctypes as C
    import torch
    lq, N, engine = env
    from paper_2404_08867_b200.configs import make_config
    from paper_2404_08867_b200.distributed import shard_range
    monkeypatch.delenv("LQ_ORBIT", raising=False)
    cfg = make_config(5)
    f = lq.parse(cfg.text, cfg.d)
    n = 1 << 26
    rule = lq.korobov_vector((cfg.plain_a | 1) % n, n, cfg.d)
    pi = engine.plain_integrand(f, cfg.d)
    z = rule.z_reduced_array()
    lay = N.lattice_layout(pi.struct, n, z)
    assert lay.mode == N.LAYOUT_ORBIT_POW2 and lay.n_supers >= 3
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


@pytest.mark.parametrize("layout", ["orbit", "paired"])
@pytest.mark.parametrize("family,scale,offset", [("expabs", 10.0, 0.0), ("expabs", 350.0, 0.0), ("expabs", 800.0, 0.0),
                                                 ("exp", 3.0, 0.25), ("exp", 100.0, -650.0), ("sincos", 9.0, 0.0)])
def test_pair_fast_direct_kernels(env, layout, family, scale, offset, monkeypatch):
    # the one-reduction point/mirror outer inlined in the
    # direct orbit kernel and the mirror-paired index kernel, against the
    # two-evaluation form (LQ_PAIRFAST=0) and the oracle; expabs 800 and the
    # exp offset -650 leave the normal range and fall back
    lq, N, engine = env
    from oracle import np_oracle
    n, d = 100003, 40
    rng = np.random.default_rng(zlib.crc32(f"pairdirect/{family}/{scale}".encode()))
    text = _pair_text(family, d, rng, scale, offset)
    f = lq.parse(text, d)
    if layout == "orbit":
        rule = lq.korobov_vector(2, n, d)
        want = N.LAYOUT_ORBIT
    else:
        rule = lq.LatticeRule(n, _unit_vector(n, d, rng))
        want = N.LAYOUT_PAIRED
    pi = engine.plain_integrand(f, d)
    z = rule.z_reduced_array()
    monkeypatch.setenv("LQ_FFT", "0")
    assert N.lattice_layout(pi.struct, n, z).mode == want
    fast = engine.lattice_sum(pi, n, z)
    monkeypatch.setenv("LQ_PAIRFAST", "0")
    slow = engine.lattice_sum(pi, n, z)
    assert math.isclose(fast, slow, rel_tol=1e-13, abs_tol=1e-300), (fast, slow)
    ref = np_oracle.slr_sum(text, n, list(rule.z_reduced))
    assert math.isclose(fast, ref, rel_tol=1e-10, abs_tol=1e-300), (fast, ref)
