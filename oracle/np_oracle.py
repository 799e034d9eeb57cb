"""Numpy restatement of the reference hot path (CPU ORACLE, test-only).

Each function cites the reference code it restates
(/root/reference/pkg/src/latquad/...).  Integrands are source text in the
reference's language, evaluated by the oracle's own literal evaluator
(``oracle/np_expr.py``): nothing here imports the product package.
"""

from __future__ import annotations

import math

import numpy as np

from oracle import np_expr

_MAX_ENUM = 2**53


def points_block(n, z, start, stop):
    """lattice.py:96-105: ((j * z_j) % n) / n in int64 then true division.
    z are the unreduced components; reduced here as z_reduced does (lattice.py:76-78)."""
    if n > _MAX_ENUM:
        raise OverflowError(f"cannot enumerate points of an n={n} rule")
    j = np.arange(start, stop, dtype=np.int64)
    zr = [int(c) % n for c in z]
    out = np.empty((len(j), len(zr)))
    for col, zj in enumerate(zr):
        out[:, col] = ((j * zj) % n) / n
    return out


def eval_array(text, d, assignment):
    """exprcore.py:442-480's job -- the integrand's values over numpy columns
    -- done by the oracle's own literal evaluator (np_expr: the source text as
    written, no canonical DAG), so the oracle shares nothing with the
    product's front end."""
    if not isinstance(text, str):
        raise TypeError("the oracle evaluates integrand source text (not a product Expr)")
    return np_expr.evaluate(text, d, assignment)


def slr_sum(f, n, z, i_begin=0, i_end=None, rows=1 << 19):
    """quad.py:96-104: per block of `rows` points, eval_array then np.sum;
    blocks accumulated in order.  Returns the raw sum (not divided by n)."""
    i_end = n if i_end is None else i_end
    d = len(z)
    acc = 0.0
    for start in range(i_begin, i_end, rows):
        stop = min(start + rows, i_end)
        pts = points_block(n, z, start, stop)
        vals = eval_array(f, d, {i + 1: pts[:, i] for i in range(d)})
        acc += float(vals) * len(pts) if np.ndim(vals) == 0 else float(np.sum(vals))
    return acc


def slr_value(f, n, z):
    return slr_sum(f, n, z) / n


def mc_value(f, d, n, seed=0, rows=1 << 19):
    """quad.py:79-93: numpy default_rng(seed).random((rows, d)) blocks,
    eval_array, float(np.sum) accumulated per block, divided by n."""
    rng = np.random.default_rng(seed)
    acc, done = 0.0, 0
    while done < n:
        m = min(rows, n - done)
        pts = rng.random((m, d))
        vals = eval_array(f, d, {i + 1: pts[:, i] for i in range(d)})
        acc += float(vals) * m if np.ndim(vals) == 0 else float(np.sum(vals))
        done += m
    return acc / n


PCG64_MULT = 0x2360ED051FC65DA44385DF649FCCF645   # numpy's PCG_DEFAULT_MULTIPLIER_128


def pcg64_draw(state, inc, k):
    """Draw k (0-based) of numpy's PCG64 stream from (state, inc), by the affine
    jump s_k = M^(k+1) s + inc (M^k + ... + 1) and the XSL-RR output -- the
    restatement the device generator (lq_mc_sum) follows."""
    mask = (1 << 128) - 1
    A, C = 1, 0
    PA, PC = PCG64_MULT, inc
    e = k + 1
    while e:
        if e & 1:
            A, C = (PA * A) & mask, (PA * C + PC) & mask
        PA, PC = (PA * PA) & mask, (PA * PC + PC) & mask
        e >>= 1
    s = (A * state + C) & mask
    rot = s >> 122
    x = ((s >> 64) ^ s) & ((1 << 64) - 1)
    out = ((x >> rot) | (x << ((64 - rot) & 63))) & ((1 << 64) - 1)
    return (out >> 11) * (1.0 / 9007199254740992.0)


def axis_counts(n, z):
    """transform.py:76-83 on the unreduced z."""
    out = [math.lcm(z[i], z[i + 1]) // min(z[i], z[i + 1]) for i in range(len(z) - 1)]
    out.append(-(-n // z[-1]))
    return tuple(out)


def midpoint_nodes(counts):
    """transform.py:169-178: (t + 0.5) / n_i as Python floats."""
    return [np.array([(t + 0.5) / ct for t in range(ct)]) for ct in counts]


def direct_tensor_sum(f, nodes, chunk=1 << 19):
    """mdi.py:104-136: flat index decoded first-axis-fastest, chunked eval_array."""
    counts = [len(a) for a in nodes]
    total = math.prod(counts) if counts else 1
    acc = 0.0
    for start in range(0, total, chunk):
        idx = np.arange(start, min(start + chunk, total), dtype=np.int64)
        assign, rem = {}, idx
        for k, (ct, arr) in enumerate(zip(counts, nodes)):
            assign[k + 1] = arr[rem % ct]
            rem = rem // ct
        vals = eval_array(f, len(counts), assign)
        acc += float(vals) * len(idx) if np.ndim(vals) == 0 else float(np.sum(vals))
    return acc


def normalize(raw, counts):
    """mdi.py:195-203."""
    total = math.prod(counts)
    if total <= 2**53:
        return raw / total
    out = raw
    for ct in counts:
        out /= ct
    return out


def separable_log_sum(factor_fns, counts):
    """MDI-LR of a product-separable integrand prod_j phi_j(x_j): the value the
    reference's level loop produces, as
    sum_j log|S_j| with S_j = sum_t phi_j(y_t) over the midpoint nodes
    (mdi.py:152-183 collapses to this for separable forms).  Returns
    (log|raw|, sign)."""
    logs, sign = 0.0, 1.0
    for fn, ct in zip(factor_fns, counts):
        y = (np.arange(ct) + 0.5) / ct
        s = float(np.sum(fn(y)))
        logs += math.log(abs(s))
        sign *= math.copysign(1.0, s)
    return logs, sign


def expabs_grid_mean_dp(k, Q, N, alpha, kappa):
    """Exact-to-rounding mean of exp(kappa |alpha + sum_j (k_j/Q) y_j|) over the
    midpoint grid y_j in {(t+1/2)/N}, for integer k_j: L*2NQ = sum_j k_j (2t_j+1)
    is an integer, so its distribution is the convolution of the per-axis
    uniform pmfs (a dimension iteration over the distribution of the partial
    linear form).  Validation oracle for the characteristic-function MDI path
    (an extension: the reference cannot express |.|)."""
    k = [int(v) for v in k]
    size = sum(kj * (2 * N - 1) for kj in k) + 1
    pmf = np.zeros(size)
    pmf[0] = 1.0
    top = 0
    for kj in k:
        nxt = np.zeros(size)
        for t in range(N):
            off = kj * (2 * t + 1)
            nxt[off:off + top + 1] += pmf[:top + 1]
        top += kj * (2 * N - 1)
        pmf = nxt / N
    m = np.arange(size, dtype=np.float64)
    L = alpha + m / (2.0 * N * Q)
    return float(np.sum(pmf * np.exp(kappa * np.abs(L))))


def linear_form_grid_mean_exact(G, steps, counts, alpha=0.0):
    """Mean of G(alpha + sum_j steps_j * (t_j + 1/2)) over the midpoint grid
    t_j in [0, counts_j), with rational steps (Fractions): the multiset of
    partial linear-form values the reference's level loop carries after
    like-term collection (mdi.py:152-165 with exprcore.py:139-169, 390-402),
    built one axis at a time as {exact value: multiplicity}, then G once per
    distinct value.  Pure Python, small grids only."""
    from fractions import Fraction
    dist = {Fraction(0): 1}
    for s, n in zip(steps, counts):
        s = Fraction(s)
        nxt = {}
        for v, cnt in dist.items():
            for t in range(n):
                key = v + s * (2 * t + 1) / 2
                nxt[key] = nxt.get(key, 0) + cnt
        dist = nxt
    total = math.prod(counts)
    return math.fsum(cnt * float(G(alpha + float(v))) for v, cnt in dist.items()) / total


def linear_form_grid_mean_np(G, k_steps, counts, alpha, h):
    """Same mean for integer steps: the form is alpha + h * sum_j k_j (2 t_j + 1);
    numpy pmf convolution, for supports too large for
    ``linear_form_grid_mean_exact``."""
    lo = sum(k * (1 if k > 0 else 2 * n - 1) for k, n in zip(k_steps, counts))
    size = sum(abs(k) * 2 * (n - 1) for k, n in zip(k_steps, counts)) + 1
    pmf = np.zeros(size)
    pmf[0] = 1.0
    top = 0
    for k, n in zip(k_steps, counts):
        a = abs(k)
        nxt = np.zeros(size)
        for t in range(n):
            nxt[2 * a * t:2 * a * t + top + 1] += pmf[:top + 1]
        top += 2 * a * (n - 1)
        pmf = nxt / n
    pos = lo + np.arange(size, dtype=np.float64)
    vals = G(alpha + h * pos)
    mask = pmf > 0
    return float(np.sum(pmf[mask] * vals[mask]))
