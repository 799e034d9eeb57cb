"""GPU: deterministic reductions -- the fixed tree, run-to-run identity, and
bit-identity of sharded (multi-GPU-shaped) partials with the one-launch path.
Shards run as sequential launches on one GPU (no inter-kernel waiting)."""

import ctypes as C

import numpy as np
import pytest
import torch

from test_distributed import _tree

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    import paper_2404_08867_b200 as lq
    from paper_2404_08867_b200 import _native as N, engine
    h = N.lib()
    ctx = N.ctx(0)
    s = torch.cuda.Stream()
    torch.cuda.set_stream(s)
    N.check(h.lq_ctx_set_stream(ctx, C.c_void_p(s.cuda_stream)))
    return lq, N, engine, h, ctx


def test_reduce_tree_matches_host_restatement(env):
    lq, N, engine, h, ctx = env
    rng = np.random.default_rng(3)
    for count in (1, 5, 1024, 1025, 5000, 70000):
        v = rng.standard_normal(count) * 10.0 ** rng.integers(-5, 5, count)
        t = torch.from_numpy(v).cuda()
        out = C.c_double()
        N.check(h.lq_reduce_sum(ctx, C.c_void_p(t.data_ptr()), count, C.byref(out)))
        assert out.value == _tree(v), count


@pytest.mark.parametrize("cid,shards", [(3, 2), (5, 8)])
def test_sharded_partials_bit_identical(env, cid, shards):
    lq, N, engine, h, ctx = env
    from paper_2404_08867_b200.configs import make_config
    from paper_2404_08867_b200.distributed import shard_range
    cfg = make_config(cid)
    rule = lq.korobov_vector(cfg.plain_a, cfg.plain_n, cfg.d)
    pi = engine.plain_integrand(lq.parse(cfg.text, cfg.d), cfg.d)
    z = rule.z_reduced_array()
    S = N.lattice_layout(pi.struct, rule.n, z).n_supers
    if cid == 5:
        S_used = 16              # first 16 super-chunks (64 Mi points) keep the test short
    else:
        S_used = S
    one = torch.zeros(S, dtype=torch.float64, device="cuda")
    N.check(h.lq_lattice_partials(ctx, C.byref(pi.struct), rule.n, N.as_ptr(z), 0, S_used, C.c_void_p(one.data_ptr())))
    many = torch.zeros(S, dtype=torch.float64, device="cuda")
    for r in range(shards):
        lo, hi = shard_range(S_used, r, shards)
        if hi > lo:
            N.check(h.lq_lattice_partials(ctx, C.byref(pi.struct), rule.n, N.as_ptr(z), lo, hi,
                                          C.c_void_p(many.data_ptr() + 8 * lo)))
    torch.cuda.synchronize()
    assert torch.equal(one.view(torch.int64), many.view(torch.int64))
    if cid == 3:
        full = engine.lattice_sum(pi, rule.n, z)
        out = C.c_double()
        N.check(h.lq_reduce_sum(ctx, C.c_void_p(one.data_ptr()), S, C.byref(out)))
        assert out.value == full


def test_run_to_run_identical(env):
    lq, N, engine, h, ctx = env
    from paper_2404_08867_b200.configs import make_config
    cfg = make_config(2)
    f = lq.parse(cfg.text, cfg.d)
    rule = lq.korobov_vector(cfg.plain_a, cfg.plain_n, cfg.d)
    vals = {lq.slr_integrate(f, rule).value for _ in range(5)}
    assert len(vals) == 1
    m = {lq.mdi_lr(f, cfg.d, cfg.mdi_a, cfg.mdi_n) for _ in range(5)}
    assert len(m) == 1


def test_mdi_sharded_blocks_bit_identical(env):
    lq, N, engine, h, ctx = env
    from paper_2404_08867_b200.configs import make_config
    from paper_2404_08867_b200.transform import axis_counts
    cfg = make_config(2)
    f = lq.parse(cfg.text, cfg.d)
    counts = axis_counts(lq.korobov_vector(cfg.mdi_a, cfg.mdi_n, cfg.d))
    # larger node counts so each factor has several 256-node blocks to shard
    counts = tuple(1024 for _ in counts)
    plan = engine.separable_plan(f, counts)
    nblk = 4
    ref = np.zeros(4)
    N.check(h.lq_mdi_sum(ctx, N.as_ptr(plan.insn), plan.n_insn, C.cast(plan.factors, C.c_void_p), plan.n_factors,
                         None, 0, N.as_ptr(plan.term_ptr), N.as_ptr(plan.term_fac), N.as_ptr(plan.coef_re),
                         N.as_ptr(plan.coef_im), N.as_ptr(plan.log_extra), plan.n_terms, N.as_ptr(ref)))
    for shards in (2, 3, 4):
        part = torch.zeros(plan.n_factors * nblk * 2, dtype=torch.float64, device="cuda")
        for r in range(shards):
            N.check(h.lq_mdi_block_sums(ctx, N.as_ptr(plan.insn), plan.n_insn, C.cast(plan.factors, C.c_void_p),
                                        plan.n_factors, None, 0, r, shards, C.c_void_p(part.data_ptr())))
        out = np.zeros(4)
        N.check(h.lq_mdi_combine(ctx, C.c_void_p(part.data_ptr()), C.cast(plan.factors, C.c_void_p),
                                 plan.n_factors, nblk, N.as_ptr(plan.term_ptr), N.as_ptr(plan.term_fac),
                                 N.as_ptr(plan.coef_re), N.as_ptr(plan.coef_im), N.as_ptr(plan.log_extra),
                                 plan.n_terms, N.as_ptr(out)))
        assert np.array_equal(out, ref), shards
