"""The reference's benchmark-suite grids run through the GPU engine and
written as RunRecord CSV rows, the caller side of the path (SURVEY.md §8(f)
item 4; grids of latquad.bench.suite_specs and the skip rules of its row
runner, /root/reference/pkg/src/latquad/bench.py:104-211).

A suite is a list of (method, integrand, d, n, a) rows in the reference's
order; a row whose direct work exceeds the desk-scale caps is recorded as
"skipped(cap)" where the reference skips it, so both implementations' CSVs
line up row for row.  Sub-second rows report the median of three timings.
Figures are not rendered.
"""

from __future__ import annotations

import itertools
import math
import statistics
import sys

from . import corpus
from .cli import MDI_DIM_CAP, RunRecord, write_rows
from .lattice import korobov_vector
from .mdi import DIRECT_CAP, GridCapError
from .quad import implr_integrate, mc_integrate, mdilr_integrate, slr_integrate

__all__ = ["SUITES", "suite_specs", "run_row", "run_suite"]


def _axis(n, d):
    return int(round(n ** (1.0 / d)))


_SWEEP = (4, 6, 8, 10, 12, 14, 16)

# suite -> rows, each generator a product over (outer .. inner) loops in the
# reference's nesting order (bench.py:104-143)
_GRIDS = {
    "test1": lambda u: [(m, f, 2, n, _axis(n, 2)) for f, n, m in itertools.product(
        ("expxy", "sinsq"), (101, 501, 1001, 5001, 10001, 40001), ("mc", "slr", "implr"))],
    "test2": lambda u: [(m, f, 3, n, _axis(n, 3)) for f, n, m in itertools.product(
        ("expsum", "sinsq"), (101, 1001, 10001, 100001, 1000001, 10000001), ("slr", "implr", "mdilr"))],
    "test3": lambda u: [(m, "gaussian", d, 1 + 10 ** d, 10) for d, m in itertools.product(
        (2, 4, 6, 8, 10, 11, 12), ("slr", "implr", "mdilr"))],
    "test4": lambda u: [("mdilr", f, d, a ** d, a) for (f, a), d in itertools.product(
        (("expalt", 8), ("ratprod", 20)),
        (10, 100, 300, 500, 700, 900, 1000) if u else (10, 20, 40, 70, 100))],
    "test5": lambda u: [("mdilr", f, d, 1 + 10 ** d, a) for f, d, a in itertools.product(
        ("gaussian", "coslin", "ratprod"), (5, 10), _SWEEP)],
    "test6": lambda u: [("mdilr", f, d, 1 + a ** d, a) for f, d, a in itertools.product(
        ("gaussian", "coslin", "ratprod"), (5, 10), _SWEEP)],
    "test7": lambda u: [("mdilr", f, d, 1 + 8 ** d, 8) for f, d in itertools.product(
        ("expalt", "ratprod", "gaussian", "coslin", "expsq", "invpow"), _SWEEP)],
}
SUITES = tuple(_GRIDS)


def suite_specs(suite, unbounded=False):
    """(method, integrand, d, n, a) rows of a suite, in the reference's order."""
    grid = _GRIDS.get(suite)
    if grid is None:
        raise ValueError(f"unknown suite {suite!r}; expected one of {SUITES}")
    return grid(unbounded)


def _infeasible(method, d, n, cap, unbounded):
    """Rows the reference skips before running (bench.py:175-199); implr and
    mdilr grid caps surface as GridCapError during the run instead."""
    if method in ("mc", "slr"):
        return n > cap
    return method == "mdilr" and d > MDI_DIM_CAP and not unbounded


def _call(method, expr, d, n, a, cap, seed, ref):
    if method == "mc":
        return mc_integrate(expr, d, n, seed=seed, reference=ref)
    if method == "slr":
        return slr_integrate(expr, korobov_vector(a, n, d), reference=ref)
    if method == "implr":
        return implr_integrate(expr, d, a, n, cap=cap, reference=ref)
    if method == "mdilr":
        return mdilr_integrate(expr, d, a, n, reference=ref)
    raise ValueError(f"unknown method {method!r}")


def run_row(spec, seed=0, unbounded=False):
    """One suite row on the GPU -> RunRecord (value from the first run; the
    seconds of sub-second rows are the median of three runs)."""
    method, fid, d, n, a = spec
    ref = corpus.reference_value(fid, d)
    cap = math.inf if unbounded else DIRECT_CAP
    skipped = RunRecord(method, fid, d, n, a, reference=ref, status="skipped(cap)")
    if _infeasible(method, d, n, cap, unbounded):
        return skipped
    expr = corpus.corpus_expr(fid, d)
    try:
        first = _call(method, expr, d, n, a, cap, seed, ref)
    except GridCapError:
        return skipped
    seconds = first.seconds
    if seconds < 1.0:
        seconds = statistics.median([seconds] + [_call(method, expr, d, n, a, cap, seed, ref).seconds
                                                 for _ in range(2)])
    return RunRecord(method, fid, d, n, a, first.value, ref, first.rel_error, seconds,
                     seed if method == "mc" else None)


def run_suite(suite, out_path, seed=0, unbounded=False, figures=False, verbose=False):
    """Every row of a suite on the GPU, written to ``out_path``; returns the
    records.  ``figures`` is accepted for latquad's signature (bench.py:226);
    rendering them is out of scope (matplotlib), so it is ignored."""
    records = []
    for spec in suite_specs(suite, unbounded=unbounded):
        rec = run_row(spec, seed, unbounded)
        if verbose:
            what = rec.status if rec.rel_error is None else f"rel={rec.rel_error:.3e} t={rec.seconds:.4f}s"
            print(f"  {rec.method:6s} {rec.integrand:9s} d={rec.d:<5d} a={rec.a:<4d} {what}", file=sys.stderr)
        records.append(rec)
    write_rows(records, out_path)
    return records
