"""Multilevel dimension iteration over the improved rule's tensor grid
(drop-in for latquad.mdi, /root/reference/pkg/src/latquad/mdi.py).

The reference strips one axis per level by symbolic partial summation with
like-term collection (mdi.py:139-192).  For a separable integrand
f = sum_tau c_tau prod_j U_{tau,j}(x_j) every level multiplies the surviving
coefficient by the cluster sum S_{tau,k} = sum_t U_{tau,k}(y_t) of the axis it
removes, so the whole iteration is the product of the d per-direction cluster
sums.  The GPU forms all d cluster sums at once (one CTA per factor and node
block, ``lq_mdi_block_sums``) and combines them in log-polar form
(``lq_mdi_combine``): the levels fuse into one pass.  Integrands that are not
separable take the reference's fallback, the direct sweep over the full grid
(mdi.py:167-179), on the GPU with the same node cap.

Reported bookkeeping follows the reference: ``levels``/``base_dim`` from the
same m/order loop, GridCapError when the base sweep exceeds ``direct_cap``
(mdi.py:112-113) -- kept for drop-in error behaviour even though the GPU does
not need the base sweep -- and ``value`` is the raw grid sum.  ``level_nodes``
reports the number of per-direction cluster sums carried per level (the GPU
has no symbolic DAG).
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass

import numpy as np

from . import engine
from ._fp import blocked_const_sum, repeated_add
from .expr import as_expr, evaluate, free_vars, node_count, var_bounds
from .lattice import korobov_vector
from .transform import AxisGridSet, midpoint_grids

__all__ = ["MdiConfig", "MdiReport", "GridCapError", "BudgetExceededError", "mdi_sum", "mdi_lr",
           "direct_tensor_sum", "DIRECT_CAP", "DEFAULT_NODE_BUDGET"]

DIRECT_CAP = 10**8                 # mdi.py:38
DEFAULT_NODE_BUDGET = 200_000      # exprcore.py:59


class GridCapError(RuntimeError):
    """The requested direct sweep exceeds the configured node cap (mdi.py:44-45)."""


class BudgetExceededError(Exception):
    """The integrand does not reduce within the budget (exprcore.py:68)."""


@dataclass(frozen=True)
class MdiConfig:
    """Engine knobs with the reference's validation (mdi.py:48-76)."""

    m: int = 1
    budget: int = DEFAULT_NODE_BUDGET
    order: str = "forward"
    fallback: str = "numeric"
    direct_cap: int = DIRECT_CAP

    def __post_init__(self):
        if not 1 <= self.m <= 3:
            raise ValueError(f"m must be 1, 2, or 3, got {self.m}")
        if self.budget < 1:
            raise ValueError(f"budget must be positive, got {self.budget}")
        if self.order not in ("forward", "reverse"):
            raise ValueError(f"order must be 'forward' or 'reverse', got {self.order!r}")
        if self.fallback not in ("numeric", "error"):
            raise ValueError(f"fallback must be 'numeric' or 'error', got {self.fallback!r}")


@dataclass
class MdiReport:
    """Observability record (mdi.py:79-101) plus GPU-side extras:
    log_raw (natural log of |value|, finite even when value under/overflows),
    sign, method ('separable' | 'cores' | 'linform' | 'subgrid' | 'direct' |
    'constant' | 'characteristic'), clusters (factor count, or support size for linform)."""

    value: float
    levels: int
    base_dim: int
    level_nodes: tuple = ()
    level_seconds: tuple = ()
    base_seconds: float = 0.0
    fallback: bool = False
    det_a: float = None
    log_raw: float = None
    sign: float = None
    method: str = None
    clusters: int = 0
    log_total: float = None

    @property
    def seconds(self):
        return float(sum(self.level_seconds)) + self.base_seconds

    @property
    def mean(self):
        """Grid mean exp(log_raw - sum log n_i): finite where ``value`` (the raw
        sum, kept reference-identical) over- or underflows FP64."""
        if self.log_raw is None or self.log_total is None:
            return None
        return (self.sign or 0.0) * math.exp(self.log_raw - self.log_total)

    @property
    def log_mean(self):
        """log |grid mean| (finite even when ``mean`` underflows, e.g. config 4)."""
        if self.log_raw is None or self.log_total is None:
            return None
        return self.log_raw - self.log_total


def _const_sweep(value, counts):
    """The reference's numeric sweep of a constant: chunks of 2^19 nodes,
    acc += c * len (mdi.py:116-128), in closed form (_fp.blocked_const_sum)."""
    total = math.prod(counts) if counts else 1
    return blocked_const_sum(value, total, 1 << 19)


def _const_levels(value, counts, cfg):
    """mdi_sum of a constant exactly as the reference's loop rounds it: each
    level's partial_sum folds N copies of the constant into one
    (make_sum, exprcore.py:139-153), then the base axes are swept in chunks
    (mdi.py:167-183).  Raises GridCapError when the base sweep exceeds the cap."""
    d = len(counts)
    levels, base_axes = _level_plan(d, cfg)
    stripped = [a for a in range(1, d + 1) if a not in base_axes]
    if cfg.order == "forward":
        stripped = stripped[::-1]
    v = float(value)
    for a in stripped:
        v = repeated_add(v, counts[a - 1])
    base = [counts[a - 1] for a in base_axes]
    base_total = math.prod(base) if base else 1
    if base_total > cfg.direct_cap:
        raise GridCapError(f"direct sweep needs {base_total} evaluations, cap is {cfg.direct_cap}")
    return (_const_sweep(v, base) if base else v), levels, base_axes


def direct_tensor_sum(g, grids, cap=DIRECT_CAP, comm=None):
    """Brute-force grid sum on the GPU (mdi.py:104-136); raises past ``cap``.
    ``comm`` (distributed.Comm): flat-index tiles sharded across ranks."""
    counts = list(grids.counts)
    total = math.prod(counts) if counts else 1
    if total > cap:
        raise GridCapError(f"direct sweep needs {total} evaluations, cap is {cap}")
    e = as_expr(g)
    if not free_vars(e):
        if not counts:
            return evaluate(e, {})
        return _const_sweep(evaluate(e, {}), counts)
    return engine.tensor_sum(e, grids, comm=comm)


def _level_plan(d, cfg):
    """Levels and base axes of the reference's loop (mdi.py:146-165): strip
    m axes per level while more than 3 remain, from the end ("forward") or the
    start ("reverse")."""
    levels = -(-(d - 3) // cfg.m) if d > 3 else 0
    base = d - levels * cfg.m
    axes = list(range(1, base + 1)) if cfg.order == "forward" else list(range(d - base + 1, d + 1))
    return levels, axes


def mdi_sum(g, grids, cfg=None, comm=None):
    """Full grid sum of g by dimension iteration (mdi.py:139-192).  ``comm``
    (distributed.Comm, size > 1) shards the device work of every branch across
    ranks with one exchange; the result is the single-GPU one bit for bit.

    The collapse the reference's symbolic levels perform is taken by the first
    branch that applies (``MdiReport.method``):
      constant      -- closed form;
      characteristic-- exp-abs of a linear form past the cap (extension);
      linform       -- G(one commensurate form), or G times separable weights;
      linform2      -- G(two commensurate forms);
      separable / cores -- product-separable terms, pieces on <= 3 axes swept;
      subgrid       -- unused axes multiply a sweep of the used ones;
      terms         -- a sum whose terms collapse by different branches;
      direct        -- the full sweep (the reference's fallback), reported
                       without fallback where its levels certainly fit."""
    cfg = cfg if cfg is not None else MdiConfig()
    d = grids.d
    e = as_expr(g)
    vb = var_bounds(e)
    if vb and (vb[0] < 1 or vb[1] > d):
        extra = free_vars(e) - set(range(1, d + 1))
        raise ValueError(f"integrand uses coordinates {sorted(extra)} beyond the {d} axes")
    counts = grids.counts if isinstance(grids.counts, tuple) else tuple(grids.counts)
    levels, base_axes = _level_plan(d, cfg)
    t0 = time.perf_counter()

    if not free_vars(e):
        value, levels, base_axes = _const_levels(evaluate(e, {}), counts, cfg)
        return MdiReport(value=value, levels=levels, base_dim=len(base_axes), level_nodes=(1,) * levels,
                         level_seconds=(0.0,) * levels, base_seconds=time.perf_counter() - t0,
                         log_raw=math.log(abs(value)) if value else -math.inf,
                         sign=math.copysign(1.0, value) if value else 0.0, method="constant", clusters=0)

    midpoint = getattr(grids, "midpoint", False)
    plan = engine.separable_plan(e, counts, None if midpoint else grids.nodes)
    usable = plan.ok and (plan.n_factors + plan.n_terms) <= cfg.budget
    pure = usable and not plan.cores
    total = _total(counts)
    if not pure and midpoint:
        # non-separable integrands whose levels still collapse: exp-abs of a
        # linear form past the direct cap by its characteristic function (an
        # extension, the reference has no |.|), functions of one commensurate
        # linear form by the distribution of the partial form (lq_mdi_linform)
        if total > cfg.direct_cap and cfg.fallback == "numeric":
            rep = _characteristic(e, d, counts, levels, base_axes, t0, comm)
            if rep is not None:
                return rep
        rep = _linform(e, counts, levels, base_axes, cfg, t0, comm, weighted=not usable)
        if rep is not None:
            return rep
        if not usable:
            rep = _linform2(e, counts, levels, base_axes, cfg, t0, comm)
            if rep is not None:
                return rep
    if not usable:
        rep = _subgrid(e, grids, counts, levels, base_axes, cfg, t0, comm)
        if rep is not None:
            return rep
        rep = _term_sum(e, grids, counts, levels, base_axes, cfg, t0, comm)
        if rep is not None:
            return rep
        bounds = _level_bounds(e, counts, levels, base_axes, cfg)
        if bounds is None and cfg.fallback == "error":
            raise BudgetExceededError("integrand is not separable over the grid axes "
                                      f"(budget {cfg.budget}); no level reduction possible")
        certified = bounds is not None
        cap = cfg.direct_cap
        if certified:
            # the reference completes its levels and sweeps only its base axes
            # (mdi.py:181-183): the cap applies to those, the GPU sweeps the grid
            base_total = math.prod(counts[a - 1] for a in base_axes)
            if base_total > cfg.direct_cap:
                raise GridCapError(f"direct sweep needs {base_total} evaluations, cap is {cfg.direct_cap}")
            cap = max(cap, total)
        value = direct_tensor_sum(e, grids, cap=cap, comm=comm)
        return MdiReport(value=value, levels=levels if certified else 0,
                         base_dim=len(base_axes) if certified else d,
                         level_nodes=bounds if certified else (), level_seconds=(0.0,) * len(bounds or ()),
                         base_seconds=time.perf_counter() - t0, fallback=not certified,
                         log_raw=math.log(abs(value)) if value else -math.inf,
                         sign=math.copysign(1.0, value) if value else 0.0, method="direct")

    base_total = math.prod(counts[a - 1] for a in base_axes)
    if base_total > cfg.direct_cap:
        raise GridCapError(f"direct sweep needs {base_total} evaluations, cap is {cfg.direct_cap}")
    log_raw, sign, raw, _ = engine.mdi_separable_sum(plan, comm)
    secs = time.perf_counter() - t0
    # "cores": product terms with a non-splitting piece on <= 3 axes, swept
    # over its own sub-grid (the reference strips the other axes level by level)
    return MdiReport(value=raw, levels=levels, base_dim=len(base_axes),
                     level_nodes=(plan.n_factors,) * levels, level_seconds=(0.0,) * levels,
                     base_seconds=secs, fallback=False, log_raw=log_raw, sign=sign,
                     method="separable" if pure else "cores", clusters=plan.n_factors)


def _level_bounds(e, counts, levels, base_axes, cfg):
    """Upper bounds on the DAG sizes the reference's levels reach for e
    (mdi.py:152-165): a partial sum over N nodes is one sum of N bound copies
    of the carried expression (exprcore.py:390-402), so a level multiplies the
    node count by at most N and adds the sum node; e's own count is taken
    twice over (plus slack) for the difference between the two canonical
    forms.  The tuple, when every bound stays within cfg.budget -- then the
    reference certainly completes its levels (no fallback, no
    BudgetExceededError) and its value is the full grid sum the direct sweep
    computes; else None (the reference may fall back, as reported)."""
    if levels == 0:
        return ()
    stripped = [a for a in range(1, len(counts) + 1) if a not in base_axes]
    if cfg.order == "forward":
        stripped = stripped[::-1]
    nc = 2 * node_count(e) + 8
    out = []
    for lev in range(levels):
        for a in stripped[lev * cfg.m:(lev + 1) * cfg.m]:
            nc = counts[a - 1] * nc + 1
        if nc > cfg.budget:
            return None
        out.append(nc)
    return tuple(out)


def _term_sum(e, grids, counts, levels, base_axes, cfg, t0, comm=None):
    """A sum whose terms collapse separately (e.g. (1 + sum x)^-2 + exp(-sum
    x^2)): the reference's levels act on each term of the sum
    (exprcore.py:390-402 distributes partial_sum over a sum), so the grid mean
    is the constant plus the coefficient-weighted term means, each by its own
    branch.  None unless every term collapses without a fallback."""
    if e.op != "add" or len(e.terms) < 2 or not midpoint_of(grids):
        return None
    mean = e.val
    parts = 0
    log_total = _log_total(counts)
    for c, t in e.terms:
        if not free_vars(t):
            mean += c * evaluate(t, {})
            continue
        try:
            rep = mdi_sum(t, grids, cfg, comm)
        except (GridCapError, BudgetExceededError):
            return None
        if rep.fallback or rep.method == "direct" or rep.log_raw is None:
            return None
        if rep.log_raw > -math.inf and rep.sign:
            mean += c * rep.sign * math.exp(rep.log_raw - log_total)
        parts += 1
    if parts < 2:
        return None
    raw, log_raw, sign = _raw_from_mean(mean, counts, log_total)
    return MdiReport(value=raw, levels=levels, base_dim=len(base_axes), level_nodes=(len(e.terms),) * levels,
                     level_seconds=(0.0,) * levels, base_seconds=time.perf_counter() - t0, fallback=False,
                     log_raw=log_raw, sign=sign, method="terms", clusters=parts)


def midpoint_of(grids):
    return getattr(grids, "midpoint", False)


def _subgrid(e, grids, counts, levels, base_axes, cfg, t0, comm=None):
    """A non-separable integrand that leaves some axes unused: every level
    that strips an unused axis only multiplies the carried expression by N
    (make_sum of N equal terms, exprcore.py:139-169), so the grid sum is
    prod_{j unused} N_j times the direct sweep over the used axes alone --
    the sweep the reference's base case performs when the used axes are its
    base axes.  None when every axis is used or that sweep exceeds the cap."""
    used = free_vars(e)
    d = len(counts)
    if len(used) >= d:
        return None
    sub_counts = tuple(c if j + 1 in used else 1 for j, c in enumerate(counts))
    sub_total = math.prod(sub_counts)
    if sub_total > cfg.direct_cap:
        return None
    if getattr(grids, "midpoint", False):
        sub = AxisGridSet(None, sub_counts, grids.n, grids.z, midpoint=True)
    else:
        sub = AxisGridSet(tuple(nd if j + 1 in used else nd[:1] for j, nd in enumerate(grids.nodes)),
                          sub_counts, grids.n, grids.z)
    part = direct_tensor_sum(e, sub, cap=cfg.direct_cap, comm=comm)
    rest = math.prod(c for j, c in enumerate(counts) if j + 1 not in used)
    if part == 0.0 or not math.isfinite(part):
        raw, log_raw, sign = part * rest, (math.log(abs(part)) if part else -math.inf), \
            (math.copysign(1.0, part) if part else 0.0)
    else:
        sign = math.copysign(1.0, part)
        log_raw = math.log(abs(part)) + math.log(rest)
        raw = part * float(rest) if rest.bit_length() <= 1000 else (
            sign * math.exp(log_raw) if log_raw < 709.7 else sign * math.inf)
    return MdiReport(value=raw, levels=levels, base_dim=len(base_axes), level_nodes=(sub_total,) * levels,
                     level_seconds=(0.0,) * levels, base_seconds=time.perf_counter() - t0, fallback=False,
                     log_raw=log_raw, sign=sign, method="subgrid", clusters=sub_total)


def _linform(e, counts, levels, base_axes, cfg, t0, comm=None, weighted=True):
    """f = G(alpha + <beta, y>), or G(...) prod_j phi_j(y_j) (weighted: each
    level's nodes carry phi_j(y_t)), with commensurate steps beta_j / (2 N_j): the
    level collapse the reference's partial sums perform by like-term
    collection (each level's partial sums take the values of the partial
    linear form, exprcore.py:139-169, 390-402; mdi.py:152-165), here as the
    distribution of that linear form convolved one direction per level on the
    GPU (lq_mdi_linform), then G over its support.  None when e is not of
    this form or its support is too large."""
    plan = engine.linform_plan(e, counts)
    # the node budget bounds what a level may carry (exprcore.py:399-401); here
    # a level carries its distinct partial-form values.  A weighted form that
    # also splits into cores takes the separable combine instead (weighted=False).
    if not plan.ok or max(plan.level_support, default=1) > cfg.budget or (plan.weights is not None and not weighted):
        return None
    mean = engine.mdi_linform_mean(plan, comm=comm)
    log_total = _log_total(counts)
    if plan.weights is not None and mean != 0.0 and math.isfinite(mean):
        # weighted form: the distribution carried scaled weights (plan.log_scale)
        sign = math.copysign(1.0, mean) * plan.sign
        log_mean = math.log(abs(mean)) + plan.log_scale
        if -700.0 < log_mean < 700.0:
            raw, log_raw, sign = _raw_from_mean(sign * math.exp(log_mean), counts, log_total)
        else:
            log_raw = log_mean + log_total
            raw = sign * (math.exp(log_raw) if log_raw < 709.7 else math.inf)
    else:
        raw, log_raw, sign = _raw_from_mean(mean, counts, log_total)
    stripped = plan.level_support[:levels * cfg.m:cfg.m] if cfg.m > 1 else plan.level_support[:levels]
    return MdiReport(value=raw, levels=levels, base_dim=len(base_axes), level_nodes=tuple(stripped),
                     level_seconds=(0.0,) * levels, base_seconds=time.perf_counter() - t0, fallback=False,
                     log_raw=log_raw, sign=sign, method="linform", clusters=plan.support)


def _linform2(e, counts, levels, base_axes, cfg, t0, comm=None):
    """f = G(<beta1, y>, <beta2, y>), two commensurate forms: the reference's
    levels carry the distinct pairs of partial forms (like-term collection,
    exprcore.py:139-169); here their joint distribution, one direction per
    level (lq_mdi_linform2), then G over its support.  None when e is not of
    this form or the joint support exceeds its cap."""
    plan = engine.linform2_plan(e, counts)
    # the grid K1 x K2 over-counts the pairs a level actually reaches (both
    # forms move with the same nodes), so only the support cap applies here;
    # where the reference's levels would overflow its budget it sums the same
    # grid directly
    if not plan.ok:
        return None
    mean = engine.mdi_linform2_mean(plan, comm=comm)
    raw, log_raw, sign = _raw_from_mean(mean, counts, _log_total(counts))
    stripped = plan.level_support[:levels * cfg.m:cfg.m] if cfg.m > 1 else plan.level_support[:levels]
    return MdiReport(value=raw, levels=levels, base_dim=len(base_axes), level_nodes=tuple(stripped),
                     level_seconds=(0.0,) * levels, base_seconds=time.perf_counter() - t0, fallback=False,
                     log_raw=log_raw, sign=sign, method="linform2", clusters=plan.support)


def _raw_from_mean(mean, counts, log_total):
    """Raw grid sum from the grid mean: one rounding (mean * total) while the
    total is a double, else through logs (under/overflow like the reference's
    float sums)."""
    if mean == 0.0 or not math.isfinite(mean):
        return mean, (math.log(abs(mean)) if mean else -math.inf), math.copysign(1.0, mean) if mean else 0.0
    sign = math.copysign(1.0, mean)
    log_raw = math.log(abs(mean)) + log_total
    total = _total(counts)
    if total.bit_length() <= 1000:
        raw = mean * float(total)
    else:
        raw = sign * math.exp(log_raw) if log_raw < 709.7 else sign * math.inf
    return raw, log_raw, sign


def _characteristic(e, d, counts, levels, base_axes, t0, comm=None):
    """K exp(kappa |alpha + <beta, x>|), kappa < 0, over the midpoint grid via
    e^{-k|L|} = (1/pi) int k/(k^2 + w^2) cos(w L) dw: the grid mean becomes a
    1-D integral of products of per-direction cluster sums
    phi_j(w) = (1/N_j) sum_t e^{i w beta_j y_t}.  An extension beyond the
    reference (which has no |.|): returns None when the integrand is not of
    this form or the truncated integral cannot be certified, and the caller
    falls back to the direct sweep."""
    fam = engine.plain_family(e, d)
    if fam is None or fam.kind != "lin_expabs" or not fam.kappa < 0.0 or fam.K == 0.0:
        return None
    beta = np.asarray(fam.beta, dtype=np.float64)
    log_total = _log_total(counts)
    if not np.any(beta):
        mean = math.exp(fam.kappa * abs(fam.alpha))
    else:
        if len(counts) < 2 or _grid_facts(counts).max_count > 2**31 - 1:
            return None
        mean, tail = engine.mdi_expabs_cf(beta, counts, fam.alpha, fam.kappa, comm)
        if not (mean > 0.0) or tail > 1e-16 * mean:
            return None
    log_raw = math.log(abs(fam.K)) + math.log(mean) + log_total
    raw = math.copysign(math.exp(log_raw), fam.K) if log_raw < 709.0 else math.copysign(math.inf, fam.K)
    return MdiReport(value=raw, levels=levels, base_dim=len(base_axes), level_nodes=(d,) * levels,
                     level_seconds=(0.0,) * levels, base_seconds=time.perf_counter() - t0, fallback=False,
                     log_raw=log_raw, sign=math.copysign(1.0, fam.K), method="characteristic", clusters=d)


def _normalize(raw, counts):
    """raw / prod(counts) without overflowing float (mdi.py:195-203).  With
    power-of-two counts every division is exact while the running value stays
    normal, so a normal result equals one ldexp (the running magnitude only
    decreases); otherwise the reference's division sequence runs as is."""
    facts = _grid_facts(counts)
    if facts.total <= 2**53:
        return raw / facts.total
    if facts.shift is not None:
        out = math.ldexp(raw, -facts.shift)
        if raw == 0.0 or not math.isfinite(raw) or abs(out) >= 2.2250738585072014e-308:
            return out
    out = raw
    for ct in counts:
        out /= ct
    return out


def _det_a(rule):
    """|A| = 1/(z_1 ... z_{d-1}); 0.0 when the product overflows float (mdi.py:206-212)."""
    if rule.d <= 1:
        return 1.0
    a = getattr(rule, "_korobov_a", None)
    if a is not None:
        e = (rule.d - 1) * (rule.d - 2) // 2       # prod_{j<d-1} a^j
        if a == 1 or e == 0:
            return 1.0
        if e * math.log2(a) > 1100:
            return 0.0
        prod = a ** e
    else:
        prod = math.prod(rule.z[:-1])
    try:
        return 1.0 / float(prod)
    except OverflowError:
        return 0.0


@dataclass(frozen=True)
class _GridFacts:
    total: int          # prod(counts), exact (thousands of bits at d = 1000)
    log_total: float    # sum log n_i
    shift: int | None   # sum log2 n_i when every n_i is a power of two
    max_count: int


_facts_cache: dict = {}


def _grid_facts(counts):
    """Per-grid constants, cached by the identity of the (immutable) counts
    tuple: a cached grid set hands the same tuple to every call, so the
    1000-entry tuple is neither hashed nor walked again (MDI-LR
    time-to-solution, cfg4/cfg5)."""
    ent = _facts_cache.get(id(counts))
    if ent is not None and ent[0] is counts:
        return ent[1]
    cs = tuple(counts)
    pow2 = all(c > 0 and c & (c - 1) == 0 for c in cs)
    facts = _GridFacts(total=math.prod(cs) if cs else 1,
                       log_total=float(sum(math.log(c) for c in cs)),
                       shift=sum(c.bit_length() - 1 for c in cs) if pow2 else None,
                       max_count=max(cs) if cs else 0)
    if len(_facts_cache) >= 64:
        _facts_cache.clear()
    _facts_cache[id(counts)] = (counts, facts)
    return facts


def _log_total(counts):
    return _grid_facts(counts).log_total


def _total(counts):
    """prod(counts) as an exact integer, cached."""
    return _grid_facts(counts).total


def mdi_lr(f, d, a, n, cfg=None, rule=None, with_report=False, comm=None):
    """Improved-rule quadrature via dimension iteration (mdi.py:215-234);
    ``comm`` shards the device work across ranks (distributed.mdi_lr)."""
    cfg = cfg if cfg is not None else MdiConfig()
    if rule is None:
        rule = korobov_vector(a, n, d)
    elif rule.d != d:
        raise ValueError(f"rule dimension {rule.d} != {d}")
    grids = midpoint_grids(rule)
    report = mdi_sum(f, grids, cfg, comm)
    report.det_a = _det_a(rule)
    report.log_total = _log_total(grids.counts)
    value = _normalize(report.value, grids.counts)
    if with_report:
        return value, report
    return value
