"""Multi-GPU sharding of both hot paths: one process per GPU,
``torch.distributed`` (NCCL over NVLink) for the single exchange step.

Plain lattice sum: the index range [0, n) is cut into fixed super-chunks of
super_tiles tiles (lq_lattice_layout, include/lq.h); rank r of P owns super-chunks
[floor(r S / P), floor((r+1) S / P)) and writes their partials into its own
slots of a zero vector of length S.  One all-reduce(SUM) over disjoint slots
is exact (x + 0 = x in IEEE arithmetic) whatever order NCCL reduces in, so
every rank then holds the same vector and runs the same fixed pairwise tree:
the estimate is bit-identical for any GPU count.

MDI-LR: the node blocks of every direction's cluster sum are split across
ranks the same way (lq_mdi_block_sums shard/nshards), exchanged with one
all-reduce over disjoint slots, then combined in log-polar form on each rank.
"""

from __future__ import annotations

import ctypes as C
import time

import numpy as np

from . import _native as N, engine
from .expr import as_expr, evaluate, free_vars
from .lattice import korobov_vector
from .mdi import MdiConfig, _level_plan, _normalize, _det_a, mdi_lr as _mdi_lr_single, GridCapError
from .quad import _result
from .transform import midpoint_grids

__all__ = ["shard_range", "exchange_disjoint", "slr_integrate", "mdi_lr", "world"]


def world(group=None):
    """(rank, size) of the default (or given) process group; (0, 1) if none."""
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized():
        return 0, 1
    return dist.get_rank(group), dist.get_world_size(group)


def _bind_stream(h, ctx):
    """Order liblq's work on torch's current stream (NCCL and the partial
    buffers live there).  The legacy default stream has handle 0, which liblq
    reads as "context-owned stream", so torch work is first moved to a
    dedicated stream in that case."""
    import torch
    s = torch.cuda.current_stream()
    if s.cuda_stream == 0:
        s = torch.cuda.Stream()
        torch.cuda.set_stream(s)
    N.check(h.lq_ctx_set_stream(ctx, C.c_void_p(s.cuda_stream)))


def shard_range(n_units, rank, size):
    """Contiguous block of ``n_units`` owned by ``rank`` of ``size``."""
    return (n_units * rank) // size, (n_units * (rank + 1)) // size


def exchange_disjoint(vec, group=None):
    """All-reduce(SUM) of a vector whose slots each have exactly one non-zero
    writer: exact and order-independent.  Works on CUDA (nccl) and CPU (gloo)
    tensors; CUDA tensors on a gloo group are staged through the host."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        if vec.is_cuda and dist.get_backend(group) != "nccl":
            host = vec.cpu()
            dist.all_reduce(host, group=group)
            vec.copy_(host)
        else:
            dist.all_reduce(vec, group=group)
    return vec


def slr_integrate(f, rule, reference=None, group=None):
    """Multi-GPU plain lattice sum (same value on every rank, bit-identical
    to the single-GPU ``quad.slr_integrate`` result path)."""
    import torch
    t0 = time.perf_counter()
    e = as_expr(f)
    rank, size = world(group)
    d, n = rule.d, rule.n
    if not free_vars(e) or size == 1:
        from .quad import slr_integrate as single
        return single(e, rule, reference)
    pi = engine.plain_integrand(e, d)
    h = N.lib()
    ctx = N.ctx(torch.cuda.current_device())
    _bind_stream(h, ctx)
    z = rule.z_reduced_array()
    S = N.lattice_layout(pi.struct, n, z).n_supers
    lo, hi = shard_range(S, rank, size)
    parts = torch.zeros(S, dtype=torch.float64, device="cuda")
    if hi > lo:
        N.check(h.lq_lattice_partials(ctx, C.byref(pi.struct), n, N.as_ptr(z), lo, hi,
                                      C.c_void_p(parts.data_ptr() + 8 * lo)))
    exchange_disjoint(parts, group)
    out = C.c_double()
    N.check(h.lq_reduce_sum(ctx, C.c_void_p(parts.data_ptr()), S, C.byref(out)))
    a = rule.z[1] if d > 1 else None
    return _result("slr", out.value / n, n, d, n, a, None, t0, reference)


def mdi_lr(f, d, a, n, cfg=None, rule=None, with_report=False, group=None):
    """Multi-GPU MDI-LR: node blocks of every cluster sum sharded across ranks."""
    import torch
    rank, size = world(group)
    if size == 1:
        return _mdi_lr_single(f, d, a, n, cfg=cfg, rule=rule, with_report=with_report)
    cfg = cfg if cfg is not None else MdiConfig()
    rule = rule if rule is not None else korobov_vector(a, n, d)
    grids = midpoint_grids(rule)
    e = as_expr(f)
    plan = engine.separable_plan(e, grids.counts) if free_vars(e) else None
    if plan is None or not plan.ok:
        return _mdi_lr_single(f, d, a, n, cfg=cfg, rule=rule, with_report=with_report)
    levels, base_axes = _level_plan(d, cfg)
    base_total = int(np.prod([grids.counts[ax - 1] for ax in base_axes], dtype=object))
    if base_total > cfg.direct_cap:
        raise GridCapError(f"direct sweep needs {base_total} evaluations, cap is {cfg.direct_cap}")
    h = N.lib()
    ctx = N.ctx(torch.cuda.current_device())
    _bind_stream(h, ctx)
    nblk = max((int(plan.factors[k].count) + N.LQ_NODE_BLOCK - 1) // N.LQ_NODE_BLOCK
               for k in range(plan.n_factors))
    part = torch.zeros(plan.n_factors * nblk * 2, dtype=torch.float64, device="cuda")
    N.check(h.lq_mdi_block_sums(ctx, N.as_ptr(plan.insn), plan.n_insn, C.cast(plan.factors, C.c_void_p),
                                plan.n_factors, None, 0, rank, size, C.c_void_p(part.data_ptr())))
    exchange_disjoint(part, group)
    out = np.zeros(4)
    N.check(h.lq_mdi_combine(ctx, C.c_void_p(part.data_ptr()), C.cast(plan.factors, C.c_void_p), plan.n_factors,
                             nblk, N.as_ptr(plan.term_ptr), N.as_ptr(plan.term_fac), N.as_ptr(plan.coef_re),
                             N.as_ptr(plan.coef_im), N.as_ptr(plan.log_extra), plan.n_terms, N.as_ptr(out)))
    raw = float(out[2])
    value = _normalize(raw, grids.counts)
    if not with_report:
        return value
    from .mdi import MdiReport
    rep = MdiReport(value=raw, levels=levels, base_dim=len(base_axes), level_nodes=(plan.n_factors,) * levels,
                    level_seconds=(0.0,) * levels, fallback=False, det_a=_det_a(rule), log_raw=float(out[0]),
                    sign=float(out[1]), method="separable", clusters=plan.n_factors)
    return value, rep
