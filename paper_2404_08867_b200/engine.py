"""Host side of the GPU engine: lowered integrands -> liblq argument structs,
and the single-GPU entry points the drop-in front-ends call.

Everything here is argument packing; all arithmetic over points, nodes and
clusters runs in liblq.so (no CPU fallback).
"""

from __future__ import annotations

import ctypes as C
import math
from collections import OrderedDict

import numpy as np

from . import _native as N, jit
from .expr import UnassignedVariableError, as_expr, evaluate, free_vars
from .lower import (compile_program, linear_outer, linear_outer2, recognize_linear_program, recognize_plain,
                    separate, weighted_linear_outer)

__all__ = ["PlainIntegrand", "plain_integrand", "lattice_sum", "tensor_program", "eval_array", "SeparablePlan",
           "separable_plan", "mdi_separable_sum"]


class _LRU(OrderedDict):
    def __init__(self, cap=64):
        super().__init__()
        self.cap = cap

    def get_or(self, key, make):
        if key in self:
            self.move_to_end(key)
            return self[key]
        val = make()
        self[key] = val
        if len(self) > self.cap:
            self.popitem(last=False)
        return val


_plain_cache = _LRU()
_prog_cache = _LRU()
_sep_cache = _LRU()
_fam_cache = _LRU()


def plain_family(e, d):
    """lower.recognize_plain(e, d), cached per (expression, d)."""
    return _fam_cache.get_or((e, d), lambda: recognize_plain(e, d))


class PlainIntegrand:
    """An lq_integrand struct plus the numpy buffers it points into."""

    def __init__(self, e, d, family=None, program=None):
        self.expr, self.d = e, d
        self.family, self.program = family, program
        s = N.Integrand()
        s.d = d
        s.alpha, s.K, s.A, s.B, s.C0, s.kappa = 0.0, 1.0, 0.0, 0.0, 0.0, -1.0
        self._keep = []
        if family is not None:
            s.kind = N.FAM[family.kind]
            beta = np.ascontiguousarray(family.beta, dtype=np.float64)
            self._keep.append(beta)
            s.beta = beta.ctypes.data
            if family.gamma is not None:
                gamma = np.ascontiguousarray(family.gamma, dtype=np.float64)
                self._keep.append(gamma)
                s.gamma = gamma.ctypes.data
            s.alpha, s.K, s.A, s.B = family.alpha, family.K, family.A, family.B
            s.C0, s.kappa, s.power = family.C0, family.kappa, float(family.power)
            if family.outer is not None:
                g = np.ascontiguousarray(family.outer.insn)
                self._keep.append(g)
                s.outer.insn = g.ctypes.data
                s.outer.n_insn = len(g)
                s.outer.n_slots = family.outer.n_slots
                s.outer.result = family.outer.result
                s.outer.n_vars = family.outer.n_vars
        if program is not None:
            if family is None:
                s.kind = 0
            ins = np.ascontiguousarray(program.insn)
            self._keep.append(ins)
            s.prog.insn = ins.ctypes.data
            s.prog.n_insn = len(ins)
            s.prog.n_slots = program.n_slots
            s.prog.result = program.result
            s.prog.n_vars = program.n_vars
        self.struct = s

    @property
    def kind(self):
        return self.family.kind if self.family is not None else "program"


def plain_integrand(f, d, force_program=False):
    """Lower f for the plain lattice sum over d coordinates (cached)."""
    e = as_expr(f)

    def make():
        fam = None if force_program else (recognize_plain(e, d) or recognize_linear_program(e, d))
        prog = compile_program(e)
        return PlainIntegrand(e, d, fam, prog)

    return _plain_cache.get_or((e, d, force_program), make)


def attach_jit(pi, n):
    """Give an interpreted plain-sum integrand its NVRTC-compiled kernel when
    the full lattice is large enough to pay for the compile (jit.py).  The
    choice depends on (f, n) only -- not on the index range of the call -- so
    every rank of a sharded sum and every sub-range call of the same lattice
    run the same code."""
    interpreted = pi.family is None or pi.family.kind == "lin_prog" or n > 2**31
    if not interpreted:
        return
    n_insn = max(len(pi.program), 1)
    if interpreted and not pi.struct.prog.jit and jit.jit_wanted(int(n) * n_insn, n_insn):
        h = jit.compile_expr(pi.expr)
        if h:
            pi.struct.prog.jit = h


def lattice_sum(pi, n, z_reduced, i_begin=0, i_end=None):
    """sum_{i in [i_begin, i_end)} f(x_i) on the GPU (not divided by n)."""
    i_end = n if i_end is None else i_end
    attach_jit(pi, n)
    out = C.c_double()
    N.check(N.lib().lq_lattice_sum(N.ctx(), C.byref(pi.struct), n, N.as_ptr(z_reduced),
                                   int(i_begin), int(i_end), C.byref(out)))
    return out.value


def tensor_program(g):
    e = as_expr(g)
    return _prog_cache.get_or(e, lambda: compile_program(e))


def _tensor_program_struct(g, grids):
    prog = tensor_program(g)
    d = grids.d
    ins = np.ascontiguousarray(prog.insn)
    from . import jit
    jh = None
    # JIT choice from the whole grid (same code on every rank and sub-range)
    if jit.jit_wanted(int(grids.total) * max(len(ins), 1), max(len(ins), 1)) and d <= 128:
        jh = jit.compile_expr(as_expr(g), n_axes=max(d, 1))
    p = N.Program(ins.ctypes.data, len(ins), prog.n_slots, prog.result, prog.n_vars, jh)
    if getattr(grids, "midpoint", False):
        nodes, mid = None, 1
    else:
        nodes = np.ascontiguousarray(np.concatenate([np.asarray(nd, dtype=np.float64) for nd in grids.nodes])
                                     if d else np.zeros(1))
        mid = 0
    return ins, p, np.asarray(grids.counts, dtype=np.int64), nodes, mid


def tensor_sum(g, grids, s_begin=0, s_end=None, comm=None):
    """Direct grid sum of g (non-constant) on the GPU; flat index first-axis-fastest.
    With ``comm`` (distributed.Comm, size > 1) the tiles of the full grid are
    sharded across ranks and exchanged: bit-identical to one GPU."""
    ins, p, counts, nodes, mid = _tensor_program_struct(g, grids)
    d = grids.d
    total = int(grids.total)
    if comm is not None and comm.size > 1 and s_begin == 0 and s_end in (None, total):
        T = -(-total // N.LQ_TILE)
        lo, hi = comm.shard(T)
        tiles = comm.zeros(T)
        if hi > lo:
            N.check(N.lib().lq_tensor_partials(comm.ctx(), C.byref(p), d, N.as_ptr(counts), N.as_ptr(nodes), mid,
                                               total, lo, hi, C.c_void_p(tiles.data_ptr())))
        return comm.reduce(comm.exchange(tiles))
    s_end = total if s_end is None else s_end
    out = C.c_double()
    N.check(N.lib().lq_tensor_sum(N.ctx(), C.byref(p), d, N.as_ptr(counts), N.as_ptr(nodes), mid,
                                  int(s_begin), int(s_end), C.byref(out)))
    return out.value


def eval_array(g, assignment):
    """exprcore.eval_array (exprcore.py:442-480) on the GPU: the values of g
    with x[j] = assignment[j] (numpy arrays broadcast together, or scalars),
    evaluated row by row by the bytecode interpreter (k_prog_eval) in the
    reference's evaluation order.  A constant g returns its float value, as
    the reference does; a missing coordinate raises UnassignedVariableError."""
    e = as_expr(g)
    fv = sorted(free_vars(e))
    if not fv:
        return evaluate(e, {})
    cols = []
    for j in fv:
        if j not in assignment:
            raise UnassignedVariableError(j)
        cols.append(np.asarray(assignment[j], dtype=np.float64))
    shaped = np.broadcast_arrays(*cols)
    shape = shaped[0].shape
    m = int(np.prod(shape)) if shape else 1
    out = np.empty(m, dtype=np.float64)
    if m == 0:
        return out.reshape(shape)
    prog = tensor_program(e)
    ins = np.ascontiguousarray(prog.insn)
    p = N.Program(ins.ctypes.data, len(ins), prog.n_slots, prog.result, prog.n_vars, None)
    flat = {j: np.ascontiguousarray(a.reshape(-1)) for j, a in zip(fv, shaped)}
    table = (C.c_void_p * max(prog.n_vars, 1))()
    for j, a in flat.items():
        table[j - 1] = a.ctypes.data
    N.check(N.lib().lq_eval_array(N.ctx(), C.byref(p), table, m, 0, out.ctypes.data))
    return out.reshape(shape) if shape else float(out[0])


# ------------------------------------------------------------------ MDI-LR

CORE_MAX_AXES = 3            # coordinates a core factor may span (lower.separate)
CORE_MAX_NODES = 10**8       # sub-grid nodes a core factor may sweep (the reference's DIRECT_CAP)


class SeparablePlan:
    """Factor table + term structure of a (partially) separable integrand on
    given axis counts.  Univariate factors become per-direction cluster sums
    on the device (k_mdi_blocks); a core factor on 2-3 axes (a piece that does
    not split, e.g. exp(x1 x2)) is swept over its own sub-grid by the direct
    tensor kernel and enters the combine as a supplied cluster sum
    (LQ_FACTOR_SUPPLIED) -- what the reference's levels do when they strip
    the other axes and sweep the rest (mdi.py:152-183)."""

    def __init__(self, e, counts, nodes=None):
        terms = separate(e, max_axes=CORE_MAX_AXES)
        self.ok = terms is not None
        if not self.ok:
            return
        d = len(counts)
        insn_parts, factors, term_ptr, term_fac = [], [], [0], []
        coef_re, coef_im, log_extra = [], [], []
        off = 0
        max_slots = 1
        fac_index = {}
        node_vals = []
        if nodes is not None:
            node_offs = np.concatenate([[0], np.cumsum([len(nd) for nd in nodes])]).astype(np.int64)
            if node_offs[-1] >= 2**31:
                raise ValueError("node table too large")
            node_vals = [np.asarray(nd, dtype=np.float64) for nd in nodes]
        else:
            node_offs = None
        n_node_vals = int(node_offs[-1]) if node_offs is not None else 0
        self.cores = []        # (slot in the nodes table, Factor, sub-grid counts)
        for t in terms:
            covered = {ax for key in t.factors for ax in key}
            extra = sum(math.log(counts[ax - 1]) for ax in range(1, d + 1) if ax not in covered)
            for axes in sorted(t.factors):
                fc = t.factors[axes]
                key = (axes, fc.R, fc.P)
                idx = fac_index.get(key)
                if idx is None:
                    rec = N.Factor()
                    if len(axes) > 1:
                        sub = tuple(int(counts[j]) if j + 1 in axes else 1 for j in range(d))
                        if math.prod(sub) > CORE_MAX_NODES:
                            self.ok = False
                            return
                        rec.count = 1
                        rec.reserved = N.LQ_FACTOR_SUPPLIED
                        rec.node_off = n_node_vals
                        self.cores.append((n_node_vals, fc, sub))
                        n_node_vals += 2
                        rec.r_off = rec.r_len = rec.r_result = rec.p_off = rec.p_len = rec.p_result = 0
                    else:
                        ax = axes[0]
                        rec.count = int(counts[ax - 1])
                        rec.node_off = -1 if node_offs is None else int(node_offs[ax - 1])
                        for which, sub in (("r", fc.R), ("p", fc.P)):
                            if sub is None:
                                setattr(rec, f"{which}_off", 0)
                                setattr(rec, f"{which}_len", 0)
                                setattr(rec, f"{which}_result", 0)
                                continue
                            prog = compile_program(sub, var_map=lambda j: 0)
                            insn_parts.append(prog.insn)
                            setattr(rec, f"{which}_off", off)
                            setattr(rec, f"{which}_len", len(prog.insn))
                            setattr(rec, f"{which}_result", prog.result)
                            off += len(prog.insn)
                            max_slots = max(max_slots, prog.n_slots)
                    idx = len(factors)
                    fac_index[key] = idx
                    factors.append(rec)
                term_fac.append(idx)
            term_ptr.append(len(term_fac))
            coef_re.append(complex(t.coef).real)
            coef_im.append(complex(t.coef).imag)
            log_extra.append(extra)
        for rec in factors:
            rec.n_slots = max_slots
        from .lower import INSN_DTYPE
        if node_vals or self.cores:
            node_vals.append(np.zeros(n_node_vals - (int(node_offs[-1]) if node_offs is not None else 0)))
            self.nodes = np.ascontiguousarray(np.concatenate(node_vals))
        else:
            self.nodes = None
        self.grid_nodes = nodes
        self.core_sums_done = False
        self.insn = (np.ascontiguousarray(np.concatenate(insn_parts)) if insn_parts
                     else np.zeros(1, dtype=INSN_DTYPE))
        self.n_insn = int(off)
        self.factors = (N.Factor * max(len(factors), 1))(*factors)
        self.n_factors = len(factors)
        self.term_ptr = np.asarray(term_ptr, dtype=np.int32)
        self.term_fac = np.asarray(term_fac if term_fac else [0], dtype=np.int32)
        self.coef_re = np.asarray(coef_re, dtype=np.float64)
        self.coef_im = np.asarray(coef_im, dtype=np.float64)
        self.log_extra = np.asarray(log_extra, dtype=np.float64)
        self.n_terms = len(terms)

    def core_sums(self, comm=None):
        """Sweep every core factor over its own sub-grid (direct tensor kernel,
        sharded across ranks with ``comm``) into the supplied-sum slots."""
        if self.core_sums_done or not self.cores:
            return
        from .expr import func as _func, mul as _mul
        from .transform import AxisGridSet
        for slot, fc, sub in self.cores:
            if self.grid_nodes is None:
                grid = AxisGridSet(None, sub, None, None, midpoint=True)
            else:
                grid = AxisGridSet(tuple(nd if c > 1 else nd[:1] for nd, c in zip(self.grid_nodes, sub)),
                                   sub, None, None)
            R = fc.R if fc.R is not None else None
            if fc.P is None:
                re, im = tensor_sum(R, grid, comm=comm), 0.0
            else:
                cos_p, sin_p = _func("cos", fc.P), _func("sin", fc.P)
                re = tensor_sum(cos_p if R is None else _mul(1.0, [R, cos_p]), grid, comm=comm)
                im = tensor_sum(sin_p if R is None else _mul(1.0, [R, sin_p]), grid, comm=comm)
            self.nodes[slot], self.nodes[slot + 1] = re, im
        self.core_sums_done = True


def separable_plan(g, counts, nodes=None):
    """Factorised plan on midpoint nodes (nodes=None) or explicit per-axis node tuples."""
    e = as_expr(g)
    key = (e, tuple(counts), None if nodes is None else tuple(tuple(nd) for nd in nodes))
    return _sep_cache.get_or(key, lambda: SeparablePlan(e, counts, nodes))


def mdi_separable_sum(plan, comm=None):
    """(log|raw|, sign, raw, im) of the full-grid sum via per-direction cluster
    sums.  With ``comm`` (size > 1) the node blocks of every direction are
    sharded across ranks ("cluster range of the current coordinate", SURVEY
    §8e), exchanged once, and combined on every rank."""
    out = np.zeros(4)
    plan.core_sums(comm)
    n_nodes = 0 if plan.nodes is None else len(plan.nodes)
    if comm is not None and comm.size > 1:
        nblk = max((int(plan.factors[k].count) + N.LQ_NODE_BLOCK - 1) // N.LQ_NODE_BLOCK
                   for k in range(plan.n_factors))
        part = comm.zeros(plan.n_factors * nblk * 2)
        ctx = comm.ctx()
        N.check(N.lib().lq_mdi_block_sums(ctx, N.as_ptr(plan.insn), plan.n_insn, C.cast(plan.factors, C.c_void_p),
                                          plan.n_factors, N.as_ptr(plan.nodes), n_nodes, comm.rank, comm.size,
                                          C.c_void_p(part.data_ptr())))
        comm.exchange(part)
        N.check(N.lib().lq_mdi_combine(ctx, C.c_void_p(part.data_ptr()), C.cast(plan.factors, C.c_void_p),
                                       plan.n_factors, nblk, N.as_ptr(plan.term_ptr), N.as_ptr(plan.term_fac),
                                       N.as_ptr(plan.coef_re), N.as_ptr(plan.coef_im), N.as_ptr(plan.log_extra),
                                       plan.n_terms, N.as_ptr(out)))
        return float(out[0]), float(out[1]), float(out[2]), float(out[3])
    N.check(N.lib().lq_mdi_sum(N.ctx(), N.as_ptr(plan.insn), plan.n_insn, C.cast(plan.factors, C.c_void_p),
                               plan.n_factors, N.as_ptr(plan.nodes), n_nodes,
                               N.as_ptr(plan.term_ptr), N.as_ptr(plan.term_fac),
                               N.as_ptr(plan.coef_re), N.as_ptr(plan.coef_im), N.as_ptr(plan.log_extra),
                               plan.n_terms, N.as_ptr(out)))
    return float(out[0]), float(out[1]), float(out[2]), float(out[3])


# --------------------------------------------- MDI-LR, exp-abs-linear family

_GL16 = np.polynomial.legendre.leggauss(16)


def cf_quadrature(beta, counts, alpha, kappa):
    """Composite 16-point Gauss-Legendre nodes on [0, Omega] for the
    characteristic-function integral, plus zero-weight tail probes."""
    beta = np.asarray(beta, dtype=np.float64)
    counts = np.asarray(counts, dtype=np.float64)
    var = float(np.sum(beta * beta * (counts * counts - 1.0) / (12.0 * counts * counts)))
    sigma = math.sqrt(var)
    omega = math.sqrt(2.0 * 75.0 / var)                       # Gaussian envelope e^-75 at Omega
    mu = abs(alpha + 0.5 * float(np.sum(beta)))
    h = 0.5 * min(abs(kappa), 1.0 / sigma, math.pi / (mu + 3.0 * sigma))
    panels = max(8, int(math.ceil(omega / h)))
    x, w = _GL16
    edges = np.linspace(0.0, omega, panels + 1)
    mid = 0.5 * (edges[1:] + edges[:-1])[:, None]
    half = 0.5 * (edges[1:] - edges[:-1])[:, None]
    nodes = (mid + half * x[None, :]).ravel()
    weights = (half * w[None, :]).ravel()
    probes = omega * np.logspace(0.0, 6.0, 64)
    return nodes, weights, probes, sigma


_cf_cache = _LRU(16)
_cf_last = [None]     # (beta object, counts object, alpha, kappa, inputs) of the last call


def _cf_inputs(beta, counts, alpha, kappa):
    """Contiguous device-call inputs of mdi_expabs_cf, cached per integrand and
    grid.  A repeated call with the very same (cached) beta array and counts
    tuple skips the key -- at d = 1000 building it was a third of config 5's
    MDI-LR time-to-solution."""
    last = _cf_last[0]
    if last is not None and last[0] is beta and last[1] is counts and last[2] == alpha and last[3] == kappa:
        return last[4]
    beta_in, counts_in = beta, counts
    beta = np.ascontiguousarray(beta, dtype=np.float64)
    key = (beta.tobytes(), tuple(int(c) for c in counts), float(alpha), float(kappa))

    def make():
        nodes, weights, probes, _ = cf_quadrature(beta, counts, alpha, kappa)
        wn = np.ascontiguousarray(np.concatenate([nodes, probes]))
        ww = np.ascontiguousarray(np.concatenate([weights, np.zeros_like(probes)]))
        return beta, np.ascontiguousarray(counts, dtype=np.int32), wn, ww, len(nodes)
    out = _cf_cache.get_or(key, make)
    _cf_last[0] = (beta_in, counts_in, alpha, kappa, out)
    return out


def mdi_expabs_cf(beta, counts, alpha, kappa, comm=None):
    """E = mean over the midpoint grid of exp(kappa |alpha + <beta, y>|), kappa < 0,
    by the characteristic function on the GPU (lq_mdi_expabs).  Returns
    (E, tail_bound) where tail_bound bounds |prod_j phi_j| beyond Omega.  With
    ``comm`` (size > 1) the frequency nodes are sharded across ranks."""
    beta, cnt, wn, ww, n_nodes = _cf_inputs(beta, counts, alpha, kappa)
    if comm is not None and comm.size > 1:
        nw = len(wn)
        buf = comm.zeros(2 * nw)
        N.check(N.lib().lq_mdi_expabs_partials(comm.ctx(), len(beta), N.as_ptr(beta), N.as_ptr(cnt), float(alpha),
                                               N.as_ptr(wn), N.as_ptr(ww), nw, float(kappa), comm.rank, comm.size,
                                               C.c_void_p(buf.data_ptr())))
        comm.exchange(buf)
        s = comm.reduce(buf, count=nw)
        logmag = buf[nw:].cpu().numpy()
        E = s * 2.0 / math.pi
        tail = float(np.exp(np.max(logmag[n_nodes:]))) if nw > n_nodes else 0.0
        return E, tail
    out = np.zeros(2)
    logmag = np.zeros(len(wn))
    N.check(N.lib().lq_mdi_expabs(N.ctx(), len(beta), N.as_ptr(beta), N.as_ptr(cnt), float(alpha),
                                  N.as_ptr(wn), N.as_ptr(ww), len(wn), float(kappa), N.as_ptr(out),
                                  N.as_ptr(logmag)))
    E = out[1] * math.exp(out[0]) * 2.0 / math.pi
    tail = float(np.exp(np.max(logmag[n_nodes:]))) if len(wn) > n_nodes else 0.0
    return E, tail


# ------------------------------- MDI-LR level collapse, G(alpha + <beta, y>)

LINFORM_MAX_SUPPORT = 1 << 28       # LQ_LINFORM_MAX_SUPPORT
LINFORM_MAX_WORK = 2 * 10**11       # sum over levels of support x nodes (~ seconds of device time)
_RATIO_DEN = 1 << 20


class LinformPlan:
    """Commensurate steps of G(<beta, y>) on the midpoint grid: direction j
    contributes beta_j (t + 1/2)/N_j = h m_j (2t + 1), so the linear form is
    h (m0 + 2k), k = sum_j |m_j| t_j (t_j uniform on [0, N_j)).  ``ok`` is
    False when the steps are not commensurate within the support cap."""

    def __init__(self, e, counts):
        from fractions import Fraction
        self.ok = False
        self.weights = None          # weighted form: axis -> phi_j Expr
        lo = linear_outer(e)
        if lo is None:
            lo = weighted_linear_outer(e)
            if lo is None:
                return
            self.weights = lo.weights
        d = len(counts)
        if self.weights is not None and any(not 1 <= j <= d for j in self.weights):
            return
        if any(not 1 <= j <= d for j in lo.beta) or not all(math.isfinite(c) for c in lo.beta.values()):
            return
        if any(int(counts[j - 1]) > LINFORM_MAX_SUPPORT for j in lo.beta):
            return                      # one axis alone would exceed the support cap
        axes = sorted(lo.beta)
        b_ref = Fraction(lo.beta[axes[0]])
        steps = []
        for j in axes:
            rho = Fraction(lo.beta[j]) / b_ref
            if rho.denominator > _RATIO_DEN:
                # a ratio within a few ulp of a small rational (e.g. 0.3 / 0.1)
                approx = rho.limit_denominator(_RATIO_DEN)
                if abs(approx - rho) > abs(rho) * Fraction(1, 1 << 50):
                    return
                rho = approx
            steps.append(rho / (2 * int(counts[j - 1])))
        den = math.lcm(*(r.denominator for r in steps))
        nums = [int(r * den) for r in steps]
        g = math.gcd(*nums)
        m = [v // g for v in nums]
        h_rat = Fraction(g, den)
        # levels in the reference's stripping order (last axis first, mdi.py:156-159)
        order = sorted(range(len(axes)), key=lambda i: -axes[i])
        self.m = np.asarray([abs(m[i]) for i in order], dtype=np.int64)
        self.n = np.asarray([int(counts[axes[i] - 1]) for i in order], dtype=np.int32)
        self.m0 = sum(mi if mi > 0 else mi * (2 * int(counts[axes[i] - 1]) - 1) for i, mi in enumerate(m))
        self.support = 1 + int(np.sum(self.m * (self.n.astype(np.int64) - 1)))
        sizes = np.cumsum(self.m * (self.n.astype(np.int64) - 1)) + 1
        work = int(np.sum(sizes * self.n))
        if self.support > LINFORM_MAX_SUPPORT or work > LINFORM_MAX_WORK:
            return
        if abs(self.m0) + 2 * self.support >= 2**53:
            return
        self.level_support = tuple(int(v) for v in sizes)
        self.wts, self.log_scale, self.sign = None, 0.0, 1.0
        if self.weights is not None and not self._node_weights(counts, [axes[i] for i in order],
                                                                [m[i] for i in order]):
            return
        self.h_exact = b_ref * h_rat                 # the quantum as an exact rational
        self.h = float(self.h_exact)
        self.G = lo.G
        self.prog = compile_program(lo.G)
        self.tiles = -(-self.support // N.LQ_TILE)
        self.ok = True

    def _node_weights(self, counts, level_axes, level_m):
        """phi_j at the midpoint nodes y_t = RN((t + 1/2)/N_j), evaluated on
        the GPU (eval_array), each axis scaled by its mean |phi_j| (the
        scales go to log_scale, so the level distributions stay O(1));
        levels with a negative step take their nodes in reverse (the plan's
        t' = N - 1 - t).  Axes weighted but outside the linear form contribute
        their scaled node mean to log_scale / sign.  False when some phi_j is
        zero or non-finite on every node."""
        per_axis = {}
        for ax, phi in self.weights.items():
            nn = int(counts[ax - 1])
            y = (np.arange(nn, dtype=np.float64) + 0.5) / nn
            with np.errstate(all="ignore"):
                v = np.asarray(eval_array(phi, {ax: y}), dtype=np.float64) * np.ones(nn)
            if not np.all(np.isfinite(v)):
                return False
            scale = float(np.mean(np.abs(v)))
            if scale == 0.0:
                return False
            per_axis[ax] = v / scale
            self.log_scale += math.log(scale)
        in_form = set(level_axes)
        for ax, v in per_axis.items():
            if ax not in in_form:
                mean = float(np.mean(v))
                if mean == 0.0:
                    return False
                self.log_scale += math.log(abs(mean))
                self.sign *= math.copysign(1.0, mean)
        cols = []
        for ax, mj in zip(level_axes, level_m):
            v = per_axis.get(ax, np.ones(int(counts[ax - 1])))
            cols.append(v[::-1] if mj < 0 else v)
        self.wts = np.ascontiguousarray(np.concatenate(cols))
        return True

    def program_struct(self):
        ins = np.ascontiguousarray(self.prog.insn)
        return ins, N.Program(ins.ctypes.data, len(ins), self.prog.n_slots, self.prog.result, self.prog.n_vars, None)


_lin_cache = _LRU(32)


def form_quantum(beta, counts):
    """Commensurate steps of one linear form on the midpoint grid: direction j
    contributes beta_j (t + 1/2)/N_j = h m_j (2t + 1) with integer m_j.
    Returns (h as an exact rational, {axis: m_j}) or None (LinformPlan's rule:
    ratios snapped to denominators <= 2^20 within 2^-50)."""
    from fractions import Fraction
    axes = sorted(beta)
    b_ref = Fraction(beta[axes[0]])
    steps = []
    for j in axes:
        rho = Fraction(beta[j]) / b_ref
        if rho.denominator > _RATIO_DEN:
            approx = rho.limit_denominator(_RATIO_DEN)
            if abs(approx - rho) > abs(rho) * Fraction(1, 1 << 50):
                return None
            rho = approx
        steps.append(rho / (2 * int(counts[j - 1])))
    den = math.lcm(*(r.denominator for r in steps))
    nums = [int(r * den) for r in steps]
    g = math.gcd(*nums)
    return b_ref * Fraction(g, den), {j: v // g for j, v in zip(axes, nums)}


LINFORM2_MAX_SUPPORT = 1 << 25     # entries of the 2-D distribution (two buffers of 256 MB)


class Linform2Plan:
    """G(<beta1, y>, <beta2, y>) with both forms commensurate: the joint
    distribution of the two partial forms, k = (sum_j |m1_j| t1_j, sum_j
    |m2_j| t2_j) with t_i = t or N - 1 - t by the sign of m_i_j, convolved one
    direction per level on a K1 x K2 grid (lq_mdi_linform2)."""

    def __init__(self, e, counts):
        self.ok = False
        lo = linear_outer2(e)
        if lo is None:
            return
        d = len(counts)
        for beta in (lo.beta1, lo.beta2):
            if any(not 1 <= j <= d for j in beta) or not all(math.isfinite(c) for c in beta.values()):
                return
        q1, q2 = form_quantum(lo.beta1, counts), form_quantum(lo.beta2, counts)
        if q1 is None or q2 is None:
            return
        (h1, m1), (h2, m2) = q1, q2
        axes = sorted(set(m1) | set(m2), reverse=True)   # the reference strips the last axis first
        self.m1 = np.asarray([m1.get(j, 0) for j in axes], dtype=np.int64)
        self.m2 = np.asarray([m2.get(j, 0) for j in axes], dtype=np.int64)
        self.n = np.asarray([int(counts[j - 1]) for j in axes], dtype=np.int32)
        nn = self.n.astype(np.int64)
        k1 = np.cumsum(np.abs(self.m1) * (nn - 1)) + 1
        k2 = np.cumsum(np.abs(self.m2) * (nn - 1)) + 1
        sizes = k1 * k2
        self.K1, self.K2 = int(k1[-1]), int(k2[-1])
        self.support = self.K1 * self.K2
        if self.support > LINFORM2_MAX_SUPPORT or int(np.sum(sizes * nn)) > LINFORM_MAX_WORK:
            return
        self.m01 = sum(v if v > 0 else v * (2 * int(counts[j - 1]) - 1) for j, v in m1.items())
        self.m02 = sum(v if v > 0 else v * (2 * int(counts[j - 1]) - 1) for j, v in m2.items())
        if max(abs(self.m01) + 2 * self.K1, abs(self.m02) + 2 * self.K2) >= 2**53:
            return
        self.level_support = tuple(int(v) for v in sizes)
        self.h1, self.h2 = float(h1), float(h2)
        self.G = lo.G
        self.prog = compile_program(lo.G)
        self.tiles = -(-self.support // N.LQ_TILE)
        self.ok = True


def linform2_plan(g, counts):
    e = as_expr(g)
    return _lin_cache.get_or((e, tuple(int(c) for c in counts), 2), lambda: Linform2Plan(e, counts))


def mdi_linform2_mean(plan, comm=None):
    """Grid mean of G(<beta1, y>, <beta2, y>) (lq_mdi_linform2); with comm
    (size > 1) the evaluation tiles of the joint support are sharded."""
    ins = np.ascontiguousarray(plan.prog.insn)
    p = N.Program(ins.ctypes.data, len(ins), plan.prog.n_slots, plan.prog.result, plan.prog.n_vars, None)
    out = C.c_double()
    args = (C.byref(p), len(plan.n), N.as_ptr(plan.m1), N.as_ptr(plan.m2), N.as_ptr(plan.n), plan.h1,
            int(plan.m01), plan.h2, int(plan.m02))
    if comm is not None and comm.size > 1:
        tiles = comm.zeros(plan.tiles)
        N.check(N.lib().lq_mdi_linform2(comm.ctx(), *args, comm.rank, comm.size, C.c_void_p(tiles.data_ptr()),
                                        plan.tiles, C.byref(out)))
        return comm.reduce(comm.exchange(tiles))
    N.check(N.lib().lq_mdi_linform2(N.ctx(), *args, 0, 1, None, plan.tiles, C.byref(out)))
    return out.value


def linform_plan(g, counts):
    """LinformPlan of g on midpoint grids with these counts (cached)."""
    e = as_expr(g)
    return _lin_cache.get_or((e, tuple(int(c) for c in counts)), lambda: LinformPlan(e, counts))


def mdi_linform_mean(plan, shard=0, nshards=1, tiles_dev=None, comm=None):
    """Grid mean of G(<beta, y>) via the level-collapse kernels (single GPU), or
    this shard's tile partials into ``tiles_dev`` (a device pointer with
    ``plan.tiles`` doubles).  With ``comm`` (size > 1): every rank convolves
    the level distributions (d small launches) and evaluates G on its share of
    the support tiles; one exchange, then the fixed tree."""
    if comm is not None and comm.size > 1:
        tiles = comm.zeros(plan.tiles)
        ins, p = plan.program_struct()
        out = C.c_double()
        N.check(N.lib().lq_mdi_linform_w(comm.ctx(), C.byref(p), len(plan.m), N.as_ptr(plan.m), N.as_ptr(plan.n),
                                         N.as_ptr(plan.wts), 0.0, plan.h, int(plan.m0), comm.rank, comm.size,
                                         C.c_void_p(tiles.data_ptr()), plan.tiles, C.byref(out)))
        return comm.reduce(comm.exchange(tiles))
    ins, p = plan.program_struct()
    out = C.c_double()
    N.check(N.lib().lq_mdi_linform_w(N.ctx(), C.byref(p), len(plan.m), N.as_ptr(plan.m), N.as_ptr(plan.n),
                                     N.as_ptr(plan.wts), 0.0, plan.h, int(plan.m0), shard, nshards,
                                     None if tiles_dev is None else C.c_void_p(tiles_dev), plan.tiles,
                                     C.byref(out)))
    return out.value
