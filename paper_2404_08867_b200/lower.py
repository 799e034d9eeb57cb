"""Expression analysis: integrand -> what the GPU runs.

Three lowerings, tried in this order by the front-ends (``quad.py``/``mdi.py``):

1. ``recognize_plain``: closed integrand families with hand-written kernels
   (exp / sin+cos / exp-abs of a linear form, exp of a diagonal quadratic).
   These are the BASELINE configs' integrands in the reference's canonical
   forms: cfg1 ``exp(sum 0.125 x_j)``, cfg2 ``A sin L + B cos L``,
   cfg3 ``K exp(sum b_j x_j + q_j x_j^2)``, cfg5 ``exp(-|sum c_j (x_j - w_j)|)``.
2. ``compile_program``: any expression as a register bytecode the generic
   CUDA interpreter evaluates per point, in the reference's evaluation order
   (sums ``v = const; v = v + c*t``, products ``v = coeff; v = v*f``;
   /root/reference/pkg/src/latquad/exprcore.py:442-480).
3. ``separate``: for MDI-LR, a factorisation f = sum_tau coef_tau prod_j
   U_{tau,j}(x_j) with complex coefficients and univariate, possibly complex
   (R(y) e^{i P(y)}) factors.  The tensor-grid sum of such a term is the
   product of per-direction cluster sums S_{tau,j} = sum_t U_{tau,j}(y_t): the
   closed form of what the reference's symbolic partial summation with
   like-term collection computes level by level (mdi.py:139-192,
   exprcore.py:139-169, 349-402).
"""

from __future__ import annotations

import cmath
import math
from dataclasses import dataclass, field

import numpy as np

from .expr import Expr, add, free_vars, func, mul, power, topo, var

__all__ = [
    "linear_form", "quad_form", "recognize_plain", "PlainFamily",
    "Program", "compile_program", "separate", "SepTerm", "Factor", "weighted_linear_outer", "WeightedOuter",
    "linear_outer2", "LinearOuter2",
    "MAX_SLOTS", "INSN_DTYPE", "LinearOuter", "linear_outer", "recognize_linear_program",
]

# ------------------------------------------------------------ polynomial view

_POLY_CAP = 4096


def _poly(e, cap=_POLY_CAP):
    """Polynomial as {monomial: coef}, monomial = ((var, power), ...) sorted;
    None if e is not a polynomial (or grows past ``cap`` monomials)."""
    memo = {}
    for node in topo(e):
        op = node.op
        if op == "const":
            p = {(): node.val}
        elif op == "var":
            p = {((node.idx, 1),): 1.0}
        elif op == "add":
            p = {(): node.val} if node.val != 0.0 else {}
            for c, t in node.terms:
                q = memo.get(t)
                if q is None:
                    p = None
                    break
                for m, v in q.items():
                    p[m] = p.get(m, 0.0) + c * v
                if len(p) > cap:
                    p = None
                    break
        elif op == "mul":
            p = {(): node.val}
            for f in node.args:
                q = memo.get(f)
                if q is None:
                    p = None
                    break
                p = _pmul(p, q, cap)
                if p is None:
                    break
        elif op == "pow" and node.idx >= 2:
            q = memo.get(node.args[0])
            p = {(): 1.0} if q is not None else None
            for _ in range(node.idx if q is not None else 0):
                p = _pmul(p, q, cap)
                if p is None:
                    break
        else:
            p = None
        memo[node] = p
    return memo.get(e)


def _pmul(p, q, cap):
    out = {}
    for m1, c1 in p.items():
        for m2, c2 in q.items():
            dm = dict(m1)
            for v, k in m2:
                dm[v] = dm.get(v, 0) + k
            key = tuple(sorted(dm.items()))
            out[key] = out.get(key, 0.0) + c1 * c2
            if len(out) > cap:
                return None
    return out


def linear_form(e):
    """(alpha, {j: beta_j}) if e is affine in the coordinates, else None."""
    if e.op == "add" and all(t.op == "var" for _, t in e.terms):
        beta = {}
        for c, t in e.terms:
            beta[t.idx] = beta.get(t.idx, 0.0) + c
        return e.val, beta
    p = _poly(e, cap=1 << 16)
    if p is None:
        return None
    alpha, beta = 0.0, {}
    for m, c in p.items():
        if not m:
            alpha += c
        elif len(m) == 1 and m[0][1] == 1:
            beta[m[0][0]] = beta.get(m[0][0], 0.0) + c
        elif c != 0.0:
            return None
    return alpha, beta


def quad_form(e):
    """(alpha, {j: (b_j, q_j)}) if e = alpha + sum_j b_j x_j + q_j x_j^2, else None."""
    p = _poly(e, cap=1 << 16)
    if p is None:
        return None
    alpha, coefs = 0.0, {}
    for m, c in p.items():
        if not m:
            alpha += c
            continue
        if len(m) != 1 or m[0][1] > 2:
            if c != 0.0:
                return None
            continue
        j, k = m[0]
        b, q = coefs.get(j, (0.0, 0.0))
        coefs[j] = (b + c, q) if k == 1 else (b, q + c)
    return alpha, coefs


# ------------------------------------------------------ plain-sum families

@dataclass
class PlainFamily:
    """A closed family the LIN/QUAD lattice-sum kernels evaluate.

    kind: 'lin_exp'     f = K exp(alpha + <beta, x>)
          'lin_sincos'  f = C0 + A sin(<beta, x>) + B cos(<beta, x>)
          'lin_expabs'  f = K exp(kappa |alpha + <beta, x>|)
          'lin_pow'     f = K (alpha + <beta, x>)^power, integer power
          'quad_exp'    f = K exp(alpha + sum_j beta_j x_j + gamma_j x_j^2)
          'quad_sincos' f = C0 + A sin(Q) + B cos(Q), Q = sum_j beta_j x_j + gamma_j x_j^2
          'prod_quad'   f = K prod_j ((x_j - beta_j)^2 + gamma_j)^power  (gamma_j NaN: no factor)
          'lin_prog'    f = G(<beta, x>), G any expression of one variable (``outer``:
                        its bytecode); the FFT-form chains evaluate G per linear form
    """

    kind: str
    d: int
    beta: np.ndarray
    gamma: np.ndarray = None
    alpha: float = 0.0
    K: float = 1.0
    A: float = 0.0
    B: float = 0.0
    C0: float = 0.0
    kappa: float = -1.0
    power: int = 0
    outer: object = None      # lin_prog: Program of G (variable 0 = <beta, x>)


def _vec(coefs, d):
    v = np.zeros(d)
    for j, c in coefs.items():
        if not 1 <= j <= d:
            return None
        v[j - 1] = c
    return v


def _strip_scale(e):
    if e.op == "mul" and len(e.args) == 1:
        return e.val, e.args[0]
    return 1.0, e


def _abs_affine(arg):
    """arg = a0 + kappa*|L| -> (a0, kappa, abs node) or None."""
    a0 = 0.0
    if arg.op == "add":
        if len(arg.terms) != 1:
            return None
        a0 = arg.val
        kappa, node = arg.terms[0]
    else:
        kappa, node = _strip_scale(arg)
    if node.op != "abs":
        return None
    return a0, kappa, node


def _shifted_square(base):
    """base = c0 + k (x_j + s)^2 (the parser's form of c0 + k (x_j - w)^2) ->
    (j, w, c) with the factor equal to k ((x_j - w)^2 + c), plus k; or None."""
    if base.op != "add" or len(base.terms) != 1:
        return None
    k, sq = base.terms[0]
    if sq.op != "pow" or sq.idx != 2 or k == 0.0:
        return None
    inner = sq.args[0]
    if inner.op == "var":
        j, s = inner.idx, 0.0
    elif inner.op == "add" and len(inner.terms) == 1 and inner.terms[0][0] == 1.0 and inner.terms[0][1].op == "var":
        j, s = inner.terms[0][1].idx, inner.val
    else:
        return None
    return j, -s, base.val / k, k


def _prod_family(K, factors, d):
    """K prod_j (c_j + k_j (x_j - w_j)^2)^p over distinct coordinates, every
    factor bounded away from 0 on [0, 1] (Genz product peak, config 4)."""
    if not factors:
        return None
    p = None
    w = np.zeros(d)
    c = np.full(d, np.nan)
    for fct in factors:
        base, k = (fct.args[0], fct.idx) if fct.op == "pow" else (fct, 1)
        if k == 0:
            return None
        if not free_vars(base):
            return None
        m = _shifted_square(base)
        if m is None:
            qf = quad_form(base)     # a + b x + q x^2, accepted when completing the square is benign
            if qf is None or len(qf[1]) != 1:
                return None
            (j, (b, q)), = qf[1].items()
            if q == 0.0:
                return None
            wj, cq = -b / (2.0 * q), qf[0] / q
            cj = cq - wj * wj
            if not (abs(cj) >= 1e-4 * abs(cq)):   # completing the square loses <= 1e4 ulp of c
                return None
            m = (j, wj, cj, q)
        j, wj, cj, kq = m
        if not 1 <= j <= d or not np.isnan(c[j - 1]):
            return None
        if p is None:
            p = k
        elif p != k:
            return None
        dist = max(-wj, wj - 1.0, 0.0)
        fmin, fmax = cj + dist * dist, cj + max(wj * wj, (1.0 - wj) ** 2)
        if not (fmin > 0.0) or not math.isfinite(fmax) or math.log2(fmax / fmin) > 58.0:
            return None
        w[j - 1], c[j - 1] = wj, cj
        K *= kq ** k
    if p is None or not math.isfinite(K):
        return None
    return PlainFamily("prod_quad", d, w, gamma=c, K=K, power=int(p))


def recognize_plain(e, d):
    """Match a closed family (PlainFamily) or return None."""
    if e.op == "mul" and len(e.args) > 1:
        return _prod_family(e.val, e.args, d)
    K, core = _strip_scale(e)
    if core.op == "exp":
        arg = core.args[0]
        lf = linear_form(arg)
        if lf is not None:
            beta = _vec(lf[1], d)
            if beta is not None:
                return PlainFamily("lin_exp", d, beta, alpha=lf[0], K=K)
        ab = _abs_affine(arg)
        if ab is not None:
            a0, kappa, node = ab
            lf = linear_form(node.args[0])
            if lf is not None:
                beta = _vec(lf[1], d)
                if beta is not None:
                    return PlainFamily("lin_expabs", d, beta, alpha=lf[0],
                                       K=K * math.exp(a0), kappa=kappa)
        qf = quad_form(arg)
        if qf is not None:
            b = _vec({j: v[0] for j, v in qf[1].items()}, d)
            g = _vec({j: v[1] for j, v in qf[1].items()}, d)
            if b is not None:
                return PlainFamily("quad_exp", d, b, gamma=g, alpha=qf[0], K=K)
        return None
    if core.op == "pow":
        # K (alpha + <beta, x>)^k: the reference's pow node (integer k, negative
        # k meaning 1 / b^-k; exprcore.py:466-468)
        lf = linear_form(core.args[0])
        if lf is not None and core.idx != 0:
            beta = _vec(lf[1], d)
            if beta is not None:
                return PlainFamily("lin_pow", d, beta, alpha=lf[0], K=K, power=int(core.idx))
        return _prod_family(K, (core,), d)
    # C0 + sum_k coef_k trig(alpha_k + F(x)) with one shared form F: linear
    # (lin_sincos) or diagonal quadratic (quad_sincos)
    if e.op == "add":
        terms, C0 = e.terms, e.val
    elif core.op in ("sin", "cos"):
        terms, C0 = ((K, core),), 0.0
    else:
        return None
    for form, kind in ((linear_form, "lin_sincos"), (quad_form, "quad_sincos")):
        fam = _trig_family(terms, C0, d, form, kind)
        if fam is not None:
            return fam
    return None


def recognize_linear_program(e, d, max_slots=32):
    """f = G(<beta, x>) for an expression no closed family matches (e.g.
    1/(1 + L^2), exp(-L^2) with L a full linear form, or sums of functions of
    one form): PlainFamily 'lin_prog' with G's bytecode, or None."""
    lo = linear_outer(e)
    if lo is None or len(lo.beta) < 2:
        return None
    beta = _vec(lo.beta, d)
    if beta is None:
        return None
    prog = compile_program(lo.G)
    if prog.n_slots > max_slots or prog.n_vars > 1:
        return None
    return PlainFamily("lin_prog", d, beta, outer=prog)


def _trig_family(terms, C0, d, form, kind):
    A = B = 0.0
    key0 = None
    for c, t in terms:
        s, t = _strip_scale(t)
        c *= s
        if t.op not in ("sin", "cos"):
            return None
        ff = form(t.args[0])
        if ff is None:
            return None
        al, coefs = ff
        if kind == "lin_sincos":
            beta = _vec(coefs, d)
            if beta is None:
                return None
            key = (beta, None)
        else:
            beta = _vec({j: v[0] for j, v in coefs.items()}, d)
            gamma = _vec({j: v[1] for j, v in coefs.items()}, d)
            if beta is None:
                return None
            key = (beta, gamma)
        if key0 is None:
            key0 = key
        elif not (np.array_equal(key0[0], key[0]) and
                  (key[1] is None or np.array_equal(key0[1], key[1]))):
            return None
        if t.op == "sin":   # sin(al + L) = sin al cos L + cos al sin L
            A += c * math.cos(al)
            B += c * math.sin(al)
        else:               # cos(al + L) = cos al cos L - sin al sin L
            A -= c * math.sin(al)
            B += c * math.cos(al)
    if key0 is None:
        return None
    return PlainFamily(kind, d, key0[0], gamma=key0[1], A=A, B=B, C0=C0)


# ------------------------------------------------------------------ bytecode

MAX_SLOTS = 512

OP_CONST, OP_VAR, OP_ACC_INIT, OP_ACC_ADD, OP_ACC_MUL = 0, 1, 2, 3, 4
OP_POW, OP_RPOW, OP_EXP, OP_SIN, OP_COS, OP_ABS, OP_ACC_ADDVAR = 5, 6, 7, 8, 9, 10, 11
_FUNC_OP = {"exp": OP_EXP, "sin": OP_SIN, "cos": OP_COS, "abs": OP_ABS}

# must match lq_insn in include/lq.h
INSN_DTYPE = np.dtype([("op", "<i4"), ("a", "<i4"), ("b", "<i4"), ("n", "<i4"), ("c", "<f8")])


@dataclass
class Program:
    """Register bytecode: insn[k] writes slot a; the value is slot ``result``."""

    insn: np.ndarray
    n_slots: int
    result: int
    n_vars: int

    def __len__(self):
        return len(self.insn)


def compile_program(e, var_map=None):
    """Compile e to bytecode; ``var_map`` maps coordinate index -> kernel
    variable number (default: j -> j-1)."""
    vm = var_map if var_map is not None else (lambda j: j - 1)
    uses = {}
    for node in topo(e):
        for ch in ([t for _, t in node.terms] if node.op == "add" else node.args):
            uses[ch] = uses.get(ch, 0) + 1
    out = []
    free = []
    state = {"next": 0, "max": 0}
    slot_of = {}
    left = dict(uses)

    def alloc():
        if free:
            return free.pop()
        s = state["next"]
        state["next"] += 1
        state["max"] = max(state["max"], state["next"])
        return s

    def release(node):
        left[node] -= 1
        if left[node] == 0 and node in slot_of:
            free.append(slot_of.pop(node))

    def emit(op, a, b=0, n=0, c=0.0):
        out.append((op, a, b, n, c))

    def ev(node):
        if node in slot_of:
            return slot_of[node]
        op = node.op
        if op == "const":
            s = alloc()
            emit(OP_CONST, s, c=node.val)
        elif op == "var":
            s = alloc()
            emit(OP_VAR, s, b=vm(node.idx))
        elif op == "add":
            s = alloc()
            emit(OP_ACC_INIT, s, c=node.val)
            for c, t in node.terms:
                if t.op == "var" and uses.get(t, 0) == 1:
                    emit(OP_ACC_ADDVAR, s, b=vm(t.idx), c=c)
                    left[t] -= 1
                    continue
                cs = ev(t)
                emit(OP_ACC_ADD, s, b=cs, c=c)
                release(t)
        elif op == "mul":
            s = alloc()
            emit(OP_ACC_INIT, s, c=node.val)
            for f in node.args:
                cs = ev(f)
                emit(OP_ACC_MUL, s, b=cs)
                release(f)
        elif op == "pow":
            cs = ev(node.args[0])
            s = alloc()
            if node.idx >= 2:
                emit(OP_POW, s, b=cs, n=node.idx)
            else:
                emit(OP_RPOW, s, b=cs, n=-node.idx)
            release(node.args[0])
        else:
            cs = ev(node.args[0])
            s = alloc()
            emit(_FUNC_OP[op], s, b=cs)
            release(node.args[0])
        if uses.get(node, 0) > 0:
            slot_of[node] = s
        return s

    res = ev(e)
    if state["max"] > MAX_SLOTS:
        raise ValueError(f"expression needs {state['max']} live slots (limit {MAX_SLOTS})")
    insn = np.zeros(len(out), dtype=INSN_DTYPE)
    for k, (op, a, b, n, c) in enumerate(out):
        insn[k] = (op, a, b, n, c)
    nv = max([vm(j) for j in free_vars(e)], default=-1) + 1
    return Program(insn, max(state["max"], 1), res, nv)


# --------------------------------------------------------- MDI separability

@dataclass(frozen=True)
class Factor:
    """Factor U(y) = R(y) * exp(i P(y)) of the coordinates ``axes`` (sorted,
    1-based): one axis for the per-direction cluster sums; two or three for a
    "core" -- a piece that does not split further, whose sum over its own
    sub-grid is taken directly (``separate(..., max_axes > 1)``).  R or P may
    be None (meaning 1 and 0)."""

    axes: tuple
    R: Expr = None
    P: Expr = None

    @property
    def axis(self):
        return self.axes[0]


@dataclass
class SepTerm:
    coef: complex
    factors: dict = field(default_factory=dict)   # axes tuple -> Factor, pairwise disjoint


_TERM_CAP = 1024


def _univ(e):
    fv = free_vars(e)
    return next(iter(fv)) if len(fv) == 1 else (0 if not fv else None)


def _fmul(f1, f2, axes):
    R = f1.R if f2.R is None else (f2.R if f1.R is None else mul(1.0, [f1.R, f2.R]))
    P = f1.P if f2.P is None else (f2.P if f1.P is None else add([(1.0, f1.P), (1.0, f2.P)]))
    return Factor(axes, R, P)


def _tmul(t1, t2, max_axes=1):
    """Product of two terms: factors on overlapping axes merge into one factor
    on the union; None when a union exceeds ``max_axes`` coordinates."""
    fac = dict(t1.factors)
    for key, f in t2.factors.items():
        axes = set(key)
        merged = f
        while True:
            hit = next((k for k in fac if axes & set(k)), None)
            if hit is None:
                break
            axes |= set(hit)
            merged = _fmul(fac.pop(hit), merged, ())
        if len(axes) > max_axes:
            return None
        key = tuple(sorted(axes))
        fac[key] = Factor(key, merged.R, merged.P)
    return SepTerm(t1.coef * t2.coef, fac)


def _additive_split(arg, max_axes=1):
    """arg = c + sum_G g_G(x_G) over disjoint coordinate groups of at most
    ``max_axes`` axes -> (c, {axes: g_G}); None otherwise."""
    if arg.op == "add":
        pieces = [(c, t) for c, t in arg.terms]
        c0 = arg.val
    else:
        pieces, c0 = [(1.0, arg)], 0.0
    groups = {}      # axes tuple -> [(coef, term)]
    for c, t in pieces:
        fv = free_vars(t)
        if not fv:
            from .expr import evaluate
            c0 += c * evaluate(t, {})
            continue
        axes = set(fv)
        members = [(c, t)]
        while True:
            hit = next((k for k in groups if axes & set(k)), None)
            if hit is None:
                break
            axes |= set(hit)
            members = groups.pop(hit) + members
        if len(axes) > max_axes:
            return None
        groups[tuple(sorted(axes))] = members
    return c0, {key: add(ps) for key, ps in groups.items()}


def separate(e, cap=_TERM_CAP, max_axes=1):
    """Factorise e into SepTerms, or None when e is not (finitely) separable.

    max_axes = 1: every factor is univariate (the per-direction cluster sums
    of the reference's level collapse).  max_axes > 1: a piece that does not
    split further but depends on at most ``max_axes`` coordinates becomes one
    core factor on them (e.g. exp(x1 x2) in exp(x1 x2) prod_j g(x_j))."""
    memo = {}

    def rec(node):
        hit = memo.get(node)
        if hit is not None or node in memo:
            return hit
        out = _rec(node)
        if out is None and max_axes > 1:
            fv = free_vars(node)
            if 2 <= len(fv) <= max_axes:
                key = tuple(sorted(fv))
                out = [SepTerm(1.0, {key: Factor(key, R=node)})]
        if out is not None and len(out) > cap:
            out = None
        memo[node] = out
        return out

    def _rec(node):
        ax = _univ(node)
        if ax == 0:
            from .expr import evaluate
            return [SepTerm(complex(evaluate(node, {})), {})]
        if ax is not None:
            return [SepTerm(1.0, {(ax,): Factor((ax,), R=node)})]
        op = node.op
        if op == "add":
            terms = [SepTerm(complex(node.val), {})] if node.val != 0.0 else []
            for c, t in node.terms:
                sub = rec(t)
                if sub is None:
                    return None
                terms.extend(SepTerm(c * s.coef, s.factors) for s in sub)
            return terms
        if op == "mul":
            acc = [SepTerm(complex(node.val), {})]
            for f in node.args:
                sub = rec(f)
                if sub is None:
                    return None
                acc = [_tmul(a, b, max_axes) for a in acc for b in sub]
                if any(t is None for t in acc) or len(acc) > cap:
                    return None
            return acc
        if op == "pow":
            sub = rec(node.args[0])
            if sub is None:
                return None
            k = node.idx
            if k >= 2:
                acc = [SepTerm(1.0, {})]
                for _ in range(k):
                    acc = [_tmul(a, b, max_axes) for a in acc for b in sub]
                    if any(t is None for t in acc) or len(acc) > cap:
                        return None
                return acc
            if len(sub) != 1:
                return None
            t = sub[0]
            if t.coef == 0:
                return None
            fac = {}
            for key, f in t.factors.items():
                R = power(f.R, k) if f.R is not None else None
                P = mul(float(k), [f.P]) if f.P is not None else None
                fac[key] = Factor(key, R, P)
            return [SepTerm(t.coef ** k, fac)]
        if op in ("exp", "sin", "cos"):
            sp = _additive_split(node.args[0], max_axes)
            if sp is None or not math.isfinite(sp[0]):
                return None
            c0, groups = sp
            if op == "exp":
                return [SepTerm(complex(math.exp(c0)),
                                {key: Factor(key, R=func("exp", g)) for key, g in groups.items()})]
            pos = {key: Factor(key, P=g) for key, g in groups.items()}
            neg = {key: Factor(key, P=mul(-1.0, [g])) for key, g in groups.items()}
            ep, en = cmath.exp(1j * c0), cmath.exp(-1j * c0)
            if op == "cos":   # (e^{i a} + e^{-i a}) / 2
                return [SepTerm(0.5 * ep, pos), SepTerm(0.5 * en, neg)]
            return [SepTerm(-0.5j * ep, pos), SepTerm(0.5j * en, neg)]   # (e^{ia} - e^{-ia}) / 2i
        return None

    return rec(e)


# ------------------------------------------- MDI: functions of one linear form

@dataclass
class LinearOuter:
    """e = G(<beta, x>): every coordinate enters through affine forms
    a_i + b_i <beta, x> with proportional coefficient vectors.  ``G`` is an
    Expr in var(1) standing for s = <beta, x>; ``beta`` maps axis -> coefficient."""

    G: Expr
    beta: dict


def _children_of(node):
    return [t for _, t in node.terms] if node.op == "add" else list(node.args)


def _rebuild(e, repl):
    """e with the nodes of ``repl`` replaced (factories re-normalise)."""
    memo = {}
    for node in topo(e):
        if node in repl:
            memo[node] = repl[node]
            continue
        op = node.op
        if op in ("const", "var"):
            out = node
        elif op == "add":
            out = add([(c, memo[t]) for c, t in node.terms], node.val)
        elif op == "mul":
            out = mul(node.val, [memo[f] for f in node.args])
        elif op == "pow":
            out = power(memo[node.args[0]], node.idx)
        else:
            out = func(op, memo[node.args[0]])
        memo[node] = out
    return memo[e]


def linear_outer(e, rel_tol=4.0 * 2.0**-52):
    """Split e = G(<beta, x>) or return None (the
    integrands whose MDI levels collapse without being separable, e.g. corpus
    invpow (1 + sum x_i)^-(d+1)).  The maximal affine subexpressions of e must
    share one coefficient direction: a_i + <beta_i, x> with beta_i = b_i beta."""
    leaves = {}
    seen = set()
    stack = [e]
    while stack:
        node = stack.pop()
        if node in seen or not free_vars(node):
            continue
        seen.add(node)
        lf = linear_form(node)
        if lf is not None:
            leaves[node] = lf
            continue
        stack.extend(_children_of(node))
    if not leaves:
        return None
    items = list(leaves.items())
    beta0 = {j: c for j, c in items[0][1][1].items() if c != 0.0}
    if not beta0:
        return None
    j0 = min(beta0)
    s = var(1)
    repl = {}
    for node, (alpha, beta) in items:
        beta = {j: c for j, c in beta.items() if c != 0.0}
        if set(beta) != set(beta0):
            return None
        b = beta[j0] / beta0[j0]
        for j, c in beta.items():
            if abs(c - b * beta0[j]) > rel_tol * abs(c):
                return None
        repl[node] = add([(b, s)], alpha)
    G = _rebuild(e, repl)
    if free_vars(G) != frozenset({1}):
        return None
    return LinearOuter(G, beta0)


@dataclass
class WeightedOuter:
    """e = coef * G(<beta, x>) * prod_j phi_j(x_j): the factors of a product
    that separate into one real univariate term each (the weights phi_j, one
    Expr per axis) times a function of one linear form.  ``G`` includes coef."""

    G: Expr
    beta: dict
    weights: dict


def weighted_linear_outer(e):
    """Split a product into separable real weights and a function of one
    linear form (None otherwise, or when either part is missing) -- the
    integrands whose MDI levels the reference collapses by like-term
    collection with node-dependent coefficients (exprcore.py:139-206)."""
    if e.op != "mul":
        return None
    coef = e.val
    rest, weights = [], {}
    for f in e.args:
        sep = separate(f) if len(free_vars(f)) > 0 else None
        if sep is not None and len(sep) == 1 and sep[0].coef.imag == 0.0 and \
                all(fac.P is None and len(fac.axes) == 1 and fac.R is not None for fac in sep[0].factors.values()):
            coef *= sep[0].coef.real
            for fac in sep[0].factors.values():
                weights.setdefault(fac.axis, []).append(fac.R)
        else:
            rest.append(f)
    if not rest or not weights or not math.isfinite(coef):
        return None
    lo = linear_outer(mul(coef, rest))
    if lo is None:
        return None
    return WeightedOuter(lo.G, lo.beta, {ax: mul(1.0, fs) for ax, fs in weights.items()})


@dataclass
class LinearOuter2:
    """e = G(<beta1, x>, <beta2, x>): the maximal affine subexpressions fall into
    exactly two proportionality classes.  ``G`` is an Expr in var(1), var(2)."""

    G: Expr
    beta1: dict
    beta2: dict


def linear_outer2(e, rel_tol=4.0 * 2.0**-52):
    """Split e = G(<beta1, x>, <beta2, x>) with two independent coefficient
    directions, or None (one direction: linear_outer; three or more: no
    collapse of this kind).  The reference's levels carry the pairs of
    partial forms for these (exprcore.py:139-169 collects like terms with
    equal pairs)."""
    leaves = {}
    seen = set()
    stack = [e]
    while stack:
        node = stack.pop()
        if node in seen or not free_vars(node):
            continue
        seen.add(node)
        lf = linear_form(node)
        if lf is not None:
            leaves[node] = lf
            continue
        stack.extend(_children_of(node))
    groups = []                        # [(beta_ref, var index)]
    repl = {}
    for node, (alpha, beta) in leaves.items():
        beta = {j: c for j, c in beta.items() if c != 0.0}
        if not beta:
            return None
        hit = None
        for ref, v in groups:
            if set(beta) != set(ref):
                continue
            j0 = min(ref)
            b = beta[j0] / ref[j0]
            if all(abs(c - b * ref[j]) <= rel_tol * abs(c) for j, c in beta.items()):
                hit = (b, v)
                break
        if hit is None:
            if len(groups) == 2:
                return None
            groups.append((beta, len(groups) + 1))
            hit = (1.0, len(groups))
        repl[node] = add([(hit[0], var(hit[1]))], alpha)
    if len(groups) != 2:
        return None
    G = _rebuild(e, repl)
    if free_vars(G) != frozenset({1, 2}):
        return None
    return LinearOuter2(G, groups[0][0], groups[1][0])
