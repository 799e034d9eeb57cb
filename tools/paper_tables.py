"""The paper's experiment grids (the reference's benchmark suites test1-test7,
latquad bench.py:104-143, which restate PAPER.md's tables) run on the B200
with the desk-scale caps lifted (``unbounded``): every row the reference
skips as infeasible -- SLR / Imp-LR over 10^10 - 10^12 points, MDI-LR at
d = 100 .. 1000 -- runs here.  One JSON line per row: method, integrand, d,
n, a, value (reference semantics: the raw-sum normalisation can overflow to
inf at d >= 300 exactly as latquad's does), the finite grid mean from
MdiReport.mean where it differs, the relative error of that mean against the
exact integral, and seconds (median of three below one second).  The
paper's Matlab CPU times for the rows it reports are quoted in BASELINE.md §1.

    python tools/paper_tables.py test1 test2 test3 test4 test5 test6 test7 > profiles/r02_paper_tables.jsonl
"""
import json
import math
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_08867_b200 as lq  # noqa: E402
from paper_2404_08867_b200 import corpus, suites  # noqa: E402

for suite in sys.argv[1:] or ["test3", "test4"]:
    for spec in suites.suite_specs(suite, unbounded=True):
        method, fid, d, n, a = spec
        t0 = time.perf_counter()
        rec = suites.run_row(spec, unbounded=True)
        row = {"suite": suite, "method": method, "integrand": fid, "d": d, "n": str(n), "a": a,
               "value": rec.value, "rel_error": rec.rel_error, "seconds": rec.seconds, "status": rec.status}
        if method == "mdilr" and rec.status == "ok" and not (rec.value and math.isfinite(rec.value)):
            # latquad's value over/underflows (raw sum / prod N_i); the mean does not
            expr, ref = corpus.corpus_expr(fid, d), corpus.reference_value(fid, d)
            times, rep = [], None
            for _ in range(3):
                t1 = time.perf_counter()
                _, rep = lq.mdi_lr(expr, d, a, n, with_report=True)
                times.append(time.perf_counter() - t1)
            row["mean"] = rep.mean
            row["log_mean"] = rep.log_mean
            if ref and math.isfinite(ref) and rep.log_mean is not None:
                row["rel_error_mean"] = abs(math.expm1(rep.log_mean - math.log(abs(ref))))
            row["seconds_mdi_lr"] = statistics.median(times)
        row["wall"] = round(time.perf_counter() - t0, 4)
        print(json.dumps(row), flush=True)
