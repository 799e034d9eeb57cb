"""Random integrands through mdi_lr on the GPU (whichever collapse branch each
takes) against the oracle's direct grid sum with its literal evaluator
(oracle/np_oracle.direct_tensor_sum).  Small grids (prod N_i <= 2e5);
ill-conditioned texts (double and extended precision disagreeing) skipped.
Prints mismatches and a summary with the branch counts; exit 1 on any
mismatch above 1e-10 (relative to the grid mean of |f|)."""
import math
import os
import random
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import paper_2404_08867_b200 as lq  # noqa: E402
from fuzz_texts import texts  # noqa: E402
from oracle import np_expr, np_oracle  # noqa: E402

rng = random.Random(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
cases = int(sys.argv[1]) if len(sys.argv) > 1 else 300
bad = checked = 0
methods = {}
for text in texts(rng, cases * 8):
    if checked >= cases:
        break
    d = rng.choice([2, 3, 4, 5, 6])
    a = rng.choice([3, 4, 5, 6])
    n = a ** d + rng.choice([0, 1])
    try:
        f = lq.parse(text, d)
    except Exception:
        continue
    if not lq.free_vars(f) or max(lq.free_vars(f)) > d:
        continue
    counts = lq.axis_counts(lq.korobov_vector(a, n, d))
    total = math.prod(counts)
    if total > 200_000:
        continue
    nodes = np_oracle.midpoint_nodes(counts)
    grid = np.meshgrid(*nodes, indexing="ij")
    cols = {j + 1: grid[j].reshape(-1) for j in range(d)}
    with np.errstate(all="ignore"):
        vals = np.asarray(np_expr.evaluate(text, d, cols), dtype=float) * np.ones(total)
        ext = np.asarray(np_expr.evaluate(text, d, {k: v.astype(np.longdouble) for k, v in cols.items()}),
                         dtype=np.longdouble) * np.ones(total, dtype=np.longdouble)
    if not np.all(np.isfinite(vals)) or float(np.max(np.abs(vals))) > 1e12:
        continue
    want, scale = float(np.mean(vals)), float(np.mean(np.abs(vals)))
    if abs(float(np.mean(ext)) - want) > 1e-12 * max(abs(want), scale):
        continue
    with np.errstate(all="ignore"):
        try:
            got, rep = lq.mdi_lr(f, d, a, n, with_report=True)
        except Exception as exc:
            bad += 1
            print(f"RAISED d={d} a={a} n={n}: {text[:80]!r}: {type(exc).__name__}: {exc}", flush=True)
            continue
    methods[rep.method] = methods.get(rep.method, 0) + 1
    checked += 1
    if not abs(got - want) <= 1e-10 * max(abs(want), scale, 1e-300):
        bad += 1
        print(f"MISMATCH d={d} a={a} n={n} [{rep.method}]: {text[:80]!r}: {got!r} vs {want!r}", flush=True)
print(f"{checked} cases, {bad} mismatches, branches {methods}")
sys.exit(1 if bad else 0)
