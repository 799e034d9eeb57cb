"""FFT form of the Korobov chain sums (k_orbit_fft) against
the direct orbit kernel and the reference's own sums, frozen per case in the
build container (tests/golden/fft.json; no FFT-kernel assertion
compares only GPU against GPU).  The correlation through an FFT is
exact up to rounding (~1e-14 relative on the linear forms), so sums agree with
the direct kernels to 1e-12 and with the oracle to the north-star 1e-10."""

import math
import os

import pytest

import fft_cases
from conftest import load_golden, unhex

pytestmark = pytest.mark.gpu

_FROZEN = {}

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


def _ref_sum(key):
    """The reference's own sum for this case, frozen in the build container
    (tests/golden/make_golden.py --only fft: latquad slr_integrate, or the
    reference's points_block + numpy for |.|, which its grammar lacks)."""
    if not _FROZEN:
        _FROZEN.update({c["key"]: c for c in load_golden("fft")})
    hit = _FROZEN.get(key)
    assert hit is not None, f"no frozen reference sum for {key}; rerun make_golden.py --only fft"
    return unhex(hit["value"]) * hit["n"]


@pytest.mark.parametrize("family", fft_cases.FAMILIES)
@pytest.mark.parametrize("n,d,kind", fft_cases.MAIN)
def test_fft_matches_direct_orbit_and_reference(env, family, n, d, kind, monkeypatch):
    lq, N, engine = env
    key, text, _, n, a = fft_cases.main_case(family, n, d, kind)
    f = lq.parse(text, d)
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
    ref = _ref_sum(key)
    assert math.isclose(fft, ref, rel_tol=REL, abs_tol=1e-10 * n), (family, n, d, fft, ref)


CFG5_FULL = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "cfg5_full.json")


@pytest.mark.skipif(not os.path.exists(CFG5_FULL), reason="cfg5_full.json not frozen")
@pytest.mark.parametrize("fft", ["default", "0"])
def test_cfg5_full_lattice_pinned_to_reference(env, fft, monkeypatch):
    """The headline: slr_integrate over all n = 2^31 - 1 points of config 5 vs
    the sum of the reference's own points_block (lattice.py:96-105) + numpy
    exp(-|x c - c.w|) over every point (make_golden.py --only cfg5_full,
    ~70 min on 8 cores), for the default FFT-form layout and the direct
    orbit kernel (LQ_FFT=0)."""
    lq, N, engine = env
    from paper_2404_08867_b200.configs import make_config
    (case,) = load_golden("cfg5_full")
    if fft == "0":
        monkeypatch.setenv("LQ_FFT", "0")
    else:
        monkeypatch.delenv("LQ_FFT", raising=False)
    cfg = make_config(5)
    f = lq.parse(cfg.text, cfg.d)
    rule = lq.korobov_vector(cfg.plain_a, cfg.plain_n, cfg.d)
    pi = engine.plain_integrand(f, cfg.d)
    mode = N.lattice_layout(pi.struct, rule.n, rule.z_reduced_array()).mode
    assert mode == (N.LAYOUT_ORBIT_FFT if fft == "default" else N.LAYOUT_ORBIT)
    got = lq.slr_integrate(f, rule).value
    want = unhex(case["value"])
    assert abs(got - want) <= 1e-10 * want, (got, want)


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


@pytest.mark.parametrize("family,scale,offset", fft_cases.PAIR)
def test_fft_pair_fast(env, family, scale, offset, monkeypatch):
    # the one-reduction point/mirror outer (PairFast) against
    # the two-exp form and the oracle; bounds past the normal range (|y| <= 700:
    # expabs 800, exp offset -650) fall back to the two-exp form
    lq, N, engine = env
    key, text, _, n, a = fft_cases.pair_case(family, scale, offset)
    d = 150
    f = lq.parse(text, d)
    rule = lq.korobov_vector(a, n, d)
    pi = engine.plain_integrand(f, d)
    z = rule.z_reduced_array()
    monkeypatch.setenv("LQ_FFT", "always")
    assert N.lattice_layout(pi.struct, n, z).mode == N.LAYOUT_ORBIT_FFT
    fast = engine.lattice_sum(pi, n, z)
    monkeypatch.setenv("LQ_PAIRFAST", "0")
    slow = engine.lattice_sum(pi, n, z)
    assert math.isclose(fast, slow, rel_tol=1e-13, abs_tol=1e-300), (fast, slow)
    ref = _ref_sum(key)
    assert math.isclose(fast, ref, rel_tol=REL, abs_tol=1e-300), (fast, ref)


@pytest.mark.parametrize("family", fft_cases.RM_FAMILIES)
@pytest.mark.parametrize("d", fft_cases.RM_DS)
def test_fft_position_bound_boundaries(env, family, d, monkeypatch):
    """The compile-time bound RM on the positions a chain reaches (RM * 256 >=
    B = 4097 - d; RM = 16 / 13 / 13 / 12 at these d) drops the dead outputs of
    the last inverse pass: the sums must not change at the switch points."""
    lq, N, engine = env
    key, text, _, n, g = fft_cases.rm_case(family, d)
    f = lq.parse(text, d)
    rule = lq.korobov_vector(g, n, d)
    pi = engine.plain_integrand(f, d)
    got = _sums(engine, N, pi, n, rule.z_reduced_array(), monkeypatch)
    fft = got.pop(N.LAYOUT_ORBIT_FFT)
    (direct,) = got.values()
    assert math.isclose(fft, direct, rel_tol=1e-12, abs_tol=1e-12 * n), (family, d, fft, direct)
    ref = _ref_sum(key)
    assert math.isclose(fft, ref, rel_tol=REL, abs_tol=1e-10 * n), (family, d, fft, ref)


@pytest.mark.parametrize("kind,n,d", fft_cases.LINPROG)
def test_fft_program_outer_matches_index_kernel_and_reference(env, kind, n, d, monkeypatch):
    """Functions of one linear form outside the closed families (PlainFamily
    'lin_prog': 1/(1 + L^2), exp(+-L^2) of a full form, mixed trig of one
    form): the FFT-form chains with G run as bytecode, against the per-index
    bytecode kernel over the whole expression and the reference's own sum."""
    lq, N, engine = env
    key, text, _, n, a = fft_cases.linprog_case(kind, n, d)
    f = lq.parse(text, d)
    rule = lq.korobov_vector(a, n, d)
    pi = engine.plain_integrand(f, d)
    assert pi.kind == "lin_prog"
    z = rule.z_reduced_array()
    got = _sums(engine, N, pi, n, z, monkeypatch)
    assert N.LAYOUT_ORBIT_FFT in got and N.LAYOUT_INDEX in got, got.keys()
    fft, index = got[N.LAYOUT_ORBIT_FFT], got[N.LAYOUT_INDEX]
    assert math.isclose(fft, index, rel_tol=1e-12, abs_tol=1e-12 * n), (key, fft, index)
    ref = _ref_sum(key)
    assert math.isclose(fft, ref, rel_tol=REL, abs_tol=1e-10 * n), (key, fft, ref)


@pytest.mark.parametrize("seed", range(4))
def test_fft_full_size_random_multipliers(env, seed, monkeypatch):
    """Config 5's integrand on n = 2^31 - 1 with other seeded multipliers a
    (other orders and coset structures of <a>): FFT form against the direct
    orbit kernel, full lattice, 1e-12."""
    lq, N, engine = env
    from paper_2404_08867_b200.configs import make_config
    import numpy as np
    cfg = make_config(5)
    n = cfg.plain_n
    a = int(np.random.default_rng(1000 + seed).integers(2, n - 1))
    f = lq.parse(cfg.text, cfg.d)
    rule = lq.korobov_vector(a, n, cfg.d)
    pi = engine.plain_integrand(f, cfg.d)
    got = _sums(engine, N, pi, n, rule.z_reduced_array(), monkeypatch)
    fft, direct = got[N.LAYOUT_ORBIT_FFT], got[N.LAYOUT_ORBIT]
    assert math.isclose(fft, direct, rel_tol=1e-12), (a, fft, direct)
