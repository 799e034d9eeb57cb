"""Host float bookkeeping that must reproduce the reference's rounding
sequence without its loop: constant integrands, where latquad accumulates the
same float once per block of points or nodes (quad.py:100-102,
mdi.py:116-128, and make_sum's constant folding, exprcore.py:139-153)."""

from __future__ import annotations

import math
from fractions import Fraction

__all__ = ["repeated_add", "blocked_const_sum"]


def repeated_add(v, count, acc=0.0):
    """acc + v + v + ... (count float additions, each rounded to nearest even),
    in O(binades) steps: inside one binade of acc every addition moves acc by
    the same multiple of ulp(acc), so runs of additions are taken at once."""
    v = float(v)
    acc = float(acc)
    count = int(count)
    if count <= 0 or v == 0.0:
        return acc
    if not (math.isfinite(v) and math.isfinite(acc)):
        return acc + v          # inf / nan absorb every further addition
    if v < 0.0:
        return -repeated_add(-v, count, -acc)
    while count > 0:
        if acc <= 0.0 or not math.isfinite(acc) or not math.isfinite(v):
            acc += v
            count -= 1
            continue
        u = math.ulp(acc)
        boundary = 2.0 ** (math.frexp(acc)[1])          # next power of two above acc
        r = Fraction(v) / Fraction(u)
        k = math.floor(r)
        frac = r - k
        if frac == Fraction(1, 2):
            # a tie: one real step leaves acc/u even, after which every tie
            # rounds to the same even increment
            acc += v
            count -= 1
            if acc >= boundary or count == 0:
                continue
            step = k if k % 2 == 0 else k + 1
        else:
            step = k + (1 if frac > Fraction(1, 2) else 0)
        if step == 0:
            return acc                                   # v below half an ulp: acc is fixed
        delta = Fraction(step) * Fraction(u)
        # additions whose exact result stays below the binade boundary
        room = (Fraction(boundary) - Fraction(acc) - Fraction(v)) / delta
        s = min(count, math.floor(room) + 1) if room >= 0 else 0
        if s <= 0:
            acc += v
            count -= 1
            continue
        acc = float(Fraction(acc) + s * delta)
        count -= s
    return acc


def blocked_const_sum(c, total, block):
    """sum over blocks of `block` items of c * len(block), accumulated in
    block order (quad.py:100-102 for constants, mdi.py:116-128)."""
    full, rem = divmod(int(total), int(block))
    acc = repeated_add(float(c) * block, full)
    if rem:
        acc += float(c) * rem
    return acc
