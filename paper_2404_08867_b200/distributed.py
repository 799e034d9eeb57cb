"""Multi-GPU sharding of both hot paths: one process per GPU,
``torch.distributed`` (NCCL over NVLink) for the single exchange step.

Plain lattice sum: the index range [0, n) is cut into fixed super-chunks of
super_tiles tiles (lq_lattice_layout, include/lq.h); rank r of P owns super-chunks
[floor(r S / P), floor((r+1) S / P)) and writes their partials into its own
slots of a zero vector of length S.  One all-reduce(SUM) over disjoint slots
is exact (x + 0 = x in IEEE arithmetic) whatever order NCCL reduces in, so
every rank then holds the same vector and runs the same fixed pairwise tree:
the estimate is bit-identical for any GPU count.

MDI-LR: the same front-end as one GPU (mdi.mdi_lr) with a Comm: the node
blocks of every direction's cluster sum (separable), the frequency nodes of
the characteristic-function integral (exp-abs past the cap), the support
tiles of the level collapse (one commensurate linear form) and the flat-index
tiles of the direct sweep are split across ranks, exchanged with one
all-reduce over disjoint slots, and reduced by the same fixed trees.
"""

from __future__ import annotations

import ctypes as C
import time


from . import _native as N, engine
from .expr import as_expr, free_vars
from .lattice import korobov_vector
from .mdi import GridCapError, mdi_lr as _mdi_lr_single
from .quad import _result
from .transform import midpoint_grids

__all__ = ["shard_range", "exchange_disjoint", "slr_integrate", "mdi_lr", "implr_integrate", "world", "Comm"]


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
    from .quad import check_plain
    check_plain(e, rule)
    if not free_vars(e) or size == 1:
        from .quad import slr_integrate as single
        return single(e, rule, reference)
    pi = engine.plain_integrand(e, d)
    engine.attach_jit(pi, n)     # the single-GPU path's code choice, a function of (f, n)
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


class Comm:
    """The exchange step of a sharded call, for the engine (engine.py): this
    rank's share of a fixed tiling, zeroed device vectors for the partials,
    one all-reduce over disjoint slots, and liblq's fixed-tree reduction."""

    def __init__(self, group=None):
        import torch
        self.group = group
        self.rank, self.size = world(group)
        self._torch = torch
        self._ctx = None

    def ctx(self):
        if self._ctx is None:
            h = N.lib()
            self._ctx = N.ctx(self._torch.cuda.current_device())
            _bind_stream(h, self._ctx)
        return self._ctx

    def shard(self, units):
        return shard_range(units, self.rank, self.size)

    def zeros(self, count):
        self.ctx()
        return self._torch.zeros(int(count), dtype=self._torch.float64, device="cuda")

    def exchange(self, vec):
        return exchange_disjoint(vec, self.group)

    def reduce(self, vec, count=None):
        out = C.c_double()
        N.check(N.lib().lq_reduce_sum(self.ctx(), C.c_void_p(vec.data_ptr()),
                                      int(vec.numel() if count is None else count), C.byref(out)))
        return out.value


def mdi_lr(f, d, a, n, cfg=None, rule=None, with_report=False, group=None):
    """Multi-GPU MDI-LR: the single-GPU front-end (validation, branch choice,
    report) with every branch's device work sharded -- node blocks of the
    cluster sums, frequency nodes of the characteristic function, support
    tiles of the level collapse, flat-index tiles of the direct sweep -- and
    one exchange each."""
    rank, size = world(group)
    comm = Comm(group) if size > 1 else None
    return _mdi_lr_single(f, d, a, n, cfg=cfg, rule=rule, with_report=with_report, comm=comm)


def implr_integrate(f, d, a, n, cap=None, rule=None, reference=None, group=None):
    """Multi-GPU implr_integrate (quad.py:107-119): the direct sweep's tiles
    sharded across ranks."""
    from .mdi import DIRECT_CAP, direct_tensor_sum
    t0 = time.perf_counter()
    cap = DIRECT_CAP if cap is None else cap
    if rule is None:
        rule = korobov_vector(a, n, d)
    grids = midpoint_grids(rule)
    total = grids.total
    if total > cap:
        raise GridCapError(f"improved rule needs {total} direct evaluations, cap is {cap}")
    rank, size = world(group)
    value = direct_tensor_sum(f, grids, cap, comm=Comm(group) if size > 1 else None) / total
    return _result("implr", value, total, d, n, a, None, t0, reference)
