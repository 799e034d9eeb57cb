"""Random integrands (the make_golden fuzz grammar: numbers, x[..] with index
arithmetic, + - * / ^, exp/sin/cos, sum/prod) on random small lattices --
Korobov over primes, 2^k and composite n, and random z -- through
slr_integrate on the GPU against the oracle's literal evaluator
(oracle/np_expr.py).  Prints mismatches and a summary; exit 1 on any
mismatch above 1e-10 (relative to max(|sum|, sum |f|))."""
import math
import os
import random
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_08867_b200 as lq  # noqa: E402
from oracle import np_expr, np_oracle  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from fuzz_texts import texts  # noqa: E402


rng = random.Random(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
cases = int(sys.argv[1]) if len(sys.argv) > 1 else 300
bad = checked = 0
for text in texts(rng, cases * 8):
    if checked >= cases:
        break
    d = rng.choice([2, 3, 4, 6])
    try:
        f = lq.parse(text, d)
    except Exception:
        continue
    if not lq.free_vars(f) or max(lq.free_vars(f)) > d:
        continue
    n = rng.choice([1009, 4096, 3003, 65537, 2**17, 100003])
    if rng.random() < 0.7:
        a = rng.randrange(2, n)
        while math.gcd(a, n) != 1:
            a = rng.randrange(2, n)
        rule = lq.korobov_vector(a, n, d)
    else:
        rule = lq.LatticeRule(n, tuple([1] + [rng.randrange(1, n) for _ in range(d - 1)]))
    with np.errstate(all="ignore"):
        pts = np_oracle.points_block(n, list(rule.z), 0, n)
        vals = np.asarray(np_expr.evaluate(text, d, {j + 1: pts[:, j] for j in range(d)}), dtype=float) * np.ones(n)
    if not np.all(np.isfinite(vals)) or float(np.max(np.abs(vals))) > 1e12:
        continue
    want = float(np.sum(vals))
    scale = float(np.sum(np.abs(vals)))
    # ill-conditioned integrands (e.g. cos of exp of a cube: arguments ~1e22,
    # where one ulp of exp moves cos arbitrarily) are skipped -- their value
    # depends on libm's last bit, not on the kernels -- detected by evaluating
    # the same text in extended precision
    with np.errstate(all="ignore"):
        ext = np.asarray(np_expr.evaluate(text, d, {j + 1: pts[:, j].astype(np.longdouble) for j in range(d)}),
                         dtype=np.longdouble) * np.ones(n, dtype=np.longdouble)
    ext_sum = float(np.sum(ext))
    if not math.isfinite(ext_sum) or abs(ext_sum - want) > 1e-12 * max(abs(want), scale):
        continue   # double and extended precision disagree: ill-conditioned
    got = lq.slr_integrate(f, rule).value * n
    checked += 1
    if not abs(got - want) <= 1e-10 * max(abs(want), scale, 1e-300):
        bad += 1
        print(f"MISMATCH d={d} n={n} z={rule.z[:3]}..: {text[:80]!r}: {got!r} vs {want!r}", flush=True)
print(f"{checked} cases, {bad} mismatches")
sys.exit(1 if bad else 0)
