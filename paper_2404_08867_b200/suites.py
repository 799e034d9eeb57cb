"""Benchmark suites over the corpus integrands, run on the GPU engine and
written as latquad RunRecord CSV rows (the caller side of the path, SURVEY.md
§8(f) item 4; reference suite runner /root/reference/pkg/src/latquad/
bench.py:104-250).

Each suite is the reference's fixed grid of (method, integrand, d, n, a)
rows; rows whose direct work exceeds the desk-scale caps are emitted as
"skipped(cap)" exactly where the reference skips them, so the CSVs of both
implementations line up row for row and ``fit`` reads either.  Timing: the
median of three runs for sub-second rows, one run otherwise (bench.py:
159-165).  Figures are not rendered (plotting is out of scope).
"""

from __future__ import annotations

import csv
import math
import sys
from pathlib import Path

from . import corpus
from .cli import CSV_COLUMNS, MDI_DIM_CAP, RunRecord
from .lattice import korobov_vector
from .mdi import DIRECT_CAP, GridCapError
from .quad import implr_integrate, mc_integrate, mdilr_integrate, slr_integrate

__all__ = ["SUITES", "suite_specs", "run_row", "run_suite", "write_csv"]

SUITES = ("test1", "test2", "test3", "test4", "test5", "test6", "test7")

# grid parameters of the reference suites (bench.py:47-52)
_T1_NS = (101, 501, 1001, 5001, 10001, 40001)
_T2_NS = (101, 1001, 10001, 100001, 1000001, 10000001)
_SWEEP_AS = (4, 6, 8, 10, 12, 14, 16)
_T7_DS = (4, 6, 8, 10, 12, 14, 16)


def _root(n, d):
    return int(round(n ** (1.0 / d)))


def suite_specs(suite, unbounded=False):
    """(method, integrand, d, n, a) rows of a suite, in the reference's order."""
    rows = []
    if suite == "test1":        # 2-D accuracy vs n: MC, plain lattice, improved lattice
        rows = [(m, fid, 2, n, _root(n, 2)) for fid in ("expxy", "sinsq") for n in _T1_NS
                for m in ("mc", "slr", "implr")]
    elif suite == "test2":      # 3-D: plain, improved, MDI-LR
        rows = [(m, fid, 3, n, _root(n, 3)) for fid in ("expsum", "sinsq") for n in _T2_NS
                for m in ("slr", "implr", "mdilr")]
    elif suite == "test3":      # gaussian over d with n = 10^d + 1, a = 10
        rows = [(m, "gaussian", d, 1 + 10 ** d, 10) for d in (2, 4, 6, 8, 10, 11, 12)
                for m in ("slr", "implr", "mdilr")]
    elif suite == "test4":      # MDI-LR cost vs d on n = a^d
        ds = (10, 100, 300, 500, 700, 900, 1000) if unbounded else (10, 20, 40, 70, 100)
        rows = [("mdilr", fid, d, a ** d, a) for fid, a in (("expalt", 8), ("ratprod", 20)) for d in ds]
    elif suite == "test5":      # MDI-LR over a at n = 10^d + 1
        rows = [("mdilr", fid, d, 1 + 10 ** d, a) for fid in ("gaussian", "coslin", "ratprod")
                for d in (5, 10) for a in _SWEEP_AS]
    elif suite == "test6":      # MDI-LR over a at n = a^d + 1
        rows = [("mdilr", fid, d, 1 + a ** d, a) for fid in ("gaussian", "coslin", "ratprod")
                for d in (5, 10) for a in _SWEEP_AS]
    elif suite == "test7":      # MDI-LR over d at n = 8^d + 1
        rows = [("mdilr", fid, d, 1 + 8 ** d, 8)
                for fid in ("expalt", "ratprod", "gaussian", "coslin", "expsq", "invpow") for d in _T7_DS]
    else:
        raise ValueError(f"unknown suite {suite!r}; expected one of {SUITES}")
    return rows


def _median3(run, first):
    if first.seconds >= 1.0:
        return first
    secs = sorted([first.seconds, run().seconds, run().seconds])
    first.seconds = secs[1]
    return first


def run_row(spec, seed=0, unbounded=False):
    """One suite row through the GPU engine -> RunRecord (bench.py:169-211)."""
    method, fid, d, n, a = spec
    expr = corpus.corpus_expr(fid, d)
    ref = corpus.reference_value(fid, d)
    cap = math.inf if unbounded else DIRECT_CAP

    def skipped():
        return RunRecord(method=method, integrand=fid, d=d, n=n, a=a, reference=ref, status="skipped(cap)")

    if method == "mc":
        if n > cap:
            return skipped()
        run = lambda: mc_integrate(expr, d, n, seed=seed, reference=ref)   # noqa: E731
    elif method == "slr":
        if n > cap:
            return skipped()
        rule = korobov_vector(a, n, d)
        run = lambda: slr_integrate(expr, rule, reference=ref)   # noqa: E731
    elif method == "implr":
        run = lambda: implr_integrate(expr, d, a, n, cap=cap, reference=ref)   # noqa: E731
    elif method == "mdilr":
        if d > MDI_DIM_CAP and not unbounded:
            return skipped()
        run = lambda: mdilr_integrate(expr, d, a, n, reference=ref)   # noqa: E731
    else:
        raise ValueError(f"unknown method {method!r}")
    try:
        res = _median3(run, run())
    except GridCapError:
        return skipped()
    return RunRecord(method=method, integrand=fid, d=d, n=n, a=a, value=res.value, reference=ref,
                     rel_error=res.rel_error, seconds=res.seconds, seed=seed if method == "mc" else None)


def _fmt(v):
    if v is None:
        return ""
    return repr(v) if isinstance(v, float) else str(v)


def write_csv(records, path):
    path = Path(path)
    if str(path.parent) not in ("", "."):
        path.parent.mkdir(parents=True, exist_ok=True)
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(CSV_COLUMNS)
        for rec in records:
            w.writerow([_fmt(getattr(rec, k)) for k in CSV_COLUMNS])
    return path


def run_suite(suite, out_path, seed=0, unbounded=False, verbose=False):
    """Run every row of a suite on the GPU and write the CSV; returns the records."""
    records = []
    for spec in suite_specs(suite, unbounded=unbounded):
        rec = run_row(spec, seed, unbounded)
        if verbose:
            tail = rec.status if rec.rel_error is None else f"rel={rec.rel_error:.3e} t={rec.seconds:.4f}s"
            print(f"  {rec.method:6s} {rec.integrand:9s} d={rec.d:<5d} a={rec.a:<4d} {tail}", file=sys.stderr)
        records.append(rec)
    write_csv(records, out_path)
    return records
