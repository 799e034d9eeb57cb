"""Freeze golden vectors from the REFERENCE implementation (run in the build
container only; /root/reference does not exist on the GPU box).

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py [--skip-slow]

Writes points.json, slr.json, mdi.json next to this file.  Every value is
produced by calling the reference's own public API
(/root/reference/pkg/src/latquad/{lattice,quad,mdi,transform}.py) on the
seeded inputs of paper_2404_08867_b200/configs.py, except the config-5
integrand exp(-|L|), which the reference grammar cannot express
(exprcore.py:638): that sum is formed from the reference's own points_block
(lattice.py:96-105) plus a numpy restatement of the integrand, labelled
"kind": "ref_points+numpy".

Floats are stored bit-exactly: scalars as float.hex(), arrays as base64 of
little-endian float64 bytes.
"""

from __future__ import annotations

import argparse
import gc
import base64
import json
import math
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

from latquad import corpus, exprcore  # noqa: E402  (reference, read-only)
from latquad.lattice import (LatticeRule, WeightModel, cbc_construct, korobov_search,  # noqa: E402
                             korobov_vector, p_alpha, points_block, shift_avg_wce_sq)
from latquad.mdi import MdiConfig, direct_tensor_sum, mdi_lr  # noqa: E402
from latquad.quad import implr_integrate, mc_integrate, mdilr_integrate, slr_integrate  # noqa: E402
from latquad.transform import axis_counts, midpoint_grids  # noqa: E402

from paper_2404_08867_b200.configs import make_config  # noqa: E402


def b64(arr):
    return base64.b64encode(np.ascontiguousarray(arr, dtype="<f8").tobytes()).decode()


def hx(v):
    return float(v).hex()


def points_cases():
    cases = []

    def add(tag, rule, start, stop):
        pts = points_block(rule, start, stop)
        cases.append({"tag": tag, "n": str(rule.n), "z": [str(c) for c in rule.z],
                      "start": start, "stop": stop, "shape": list(pts.shape), "data": b64(pts)})

    add("four_point", LatticeRule(4, (1, 3)), 0, 4)
    add("origin", LatticeRule(1, (1, 1, 1)), 0, 1)
    add("korobov_7_81_3", korobov_vector(7, 81, 3), 0, 81)
    add("rule_101_1_40", LatticeRule(101, (1, 40)), 0, 101)
    add("korobov_10_101_3_unreduced", korobov_vector(10, 101, 3), 0, 101)
    for cid in (1, 2, 3, 5):
        cfg = make_config(cid)
        rule = LatticeRule(cfg.plain_n, cfg.plain_z())
        n = cfg.plain_n
        rows = {1: n, 2: 48, 3: 16, 5: 8}[cid]
        add(f"cfg{cid}_head", rule, 0, min(rows, n))
        if rows < n:
            add(f"cfg{cid}_tail", rule, n - rows, n)
            mid = n // 2 + 12345 % n
            add(f"cfg{cid}_mid", rule, mid, min(mid + rows, n))
    # large moduli where the reference's int64 j*z_j stays exact (j*z < 2^63)
    big = LatticeRule(2**31 + 11, (1, 2**31 - 5, 1_234_567_891, 7))
    add("n_2p31_plus", big, 2**31 + 11 - 16, 2**31 + 11)
    big2 = LatticeRule(2**33 + 17, (1, 3_000_000_019, 5))
    add("n_2p33_plus", big2, 2**30, 2**30 + 16)
    big3 = LatticeRule(2**50 + 55, (1, 977, 12_345))
    add("n_2p50_plus", big3, 2**40, 2**40 + 16)
    return cases


def slr_cases(skip_slow):
    out = []

    def add(tag, text, d, rule, kind="reference", **extra):
        f = exprcore.parse(text, d)
        t0 = time.perf_counter()
        r = slr_integrate(f, rule)
        out.append({"tag": tag, "kind": kind, "text": text, "d": d, "n": str(rule.n),
                    "z": [str(c) for c in rule.z], "value": hx(r.value),
                    "a": r.a, "ref_seconds": time.perf_counter() - t0, **extra})

    add("const_2p5", "2.5", 2, LatticeRule(101, (1, 10)))
    add("dual_mode", "cos(2*pi*(3*x[1] - x[2]))", 2, LatticeRule(8, (1, 3)))
    add("nondual_mode", "cos(2*pi*x[1])", 2, LatticeRule(8, (1, 3)))
    add("expxy_101", corpus.get("expxy").text, 2, korobov_vector(10, 101, 2))
    add("expxy_40001", corpus.get("expxy").text, 2, korobov_vector(200, 40001, 2))
    add("sinsq_2027", corpus.get("sinsq").text, 2, korobov_vector(45, 2027, 2))
    add("expsum3_1e6", corpus.get("expsum").text, 3, korobov_vector(100, 10**6 + 1, 3))
    add("gaussian5", corpus.get("gaussian").text, 5, korobov_vector(33, 4099, 5))
    add("ratprod4", corpus.get("ratprod").text, 4, korobov_vector(77, 3001, 4))
    add("invpow3", corpus.get("invpow").text, 3, korobov_vector(19, 2003, 3))
    add("expsq4", corpus.get("expsq").text, 4, korobov_vector(31, 2999, 4))
    add("coslin6", corpus.get("coslin").text, 6, korobov_vector(13, 5003, 6))
    add("expalt7", corpus.get("expalt").text, 7, korobov_vector(21, 7001, 7))
    add("poly_mix", "x[1]^3*x[2] - 0.5*x[3]^2 + x[1]*x[2]*x[3] + 0.25", 3,
        korobov_vector(5, 1021, 3))
    add("recip_sum", "1/(1 + x[1] + 2*x[2])", 2, korobov_vector(7, 997, 2))
    add("sin_of_prod", "sin(x[1]*x[2]) + exp(-x[3])*cos(3*x[1])", 3, korobov_vector(9, 1499, 3))
    for cid in (1, 2, 3):
        if cid == 3 and skip_slow:
            continue
        cfg = make_config(cid)
        add(f"cfg{cid}", cfg.text, cfg.d, LatticeRule(cfg.plain_n, cfg.plain_z()))

    # config 5: reference points + numpy restatement of exp(-|sum c_j (x_j - w_j)|)
    cfg = make_config(5)
    rule = LatticeRule(cfg.plain_n, cfg.plain_z())
    c = np.asarray(cfg.c)
    w = np.asarray(cfg.w)
    cw = float(np.dot(c, w))
    for (lo, hi) in ((0, 1 << 14), (cfg.plain_n - (1 << 12), cfg.plain_n), (1 << 30, (1 << 30) + (1 << 12))):
        pts = points_block(rule, lo, hi)
        vals = np.exp(-np.abs(pts @ c - cw))
        out.append({"tag": f"cfg5_range_{lo}_{hi}", "kind": "ref_points+numpy", "text": cfg.text,
                    "d": cfg.d, "n": str(rule.n), "z": [str(v) for v in rule.z],
                    "i_begin": lo, "i_end": hi, "range_sum": hx(float(np.sum(vals))),
                    "value": None})
    return out


def mdi_cases(skip_slow):
    out = []

    def rep_fields(rep):
        return {"raw": hx(rep.value), "levels": rep.levels, "base_dim": rep.base_dim,
                "fallback": rep.fallback, "det_a": hx(rep.det_a) if rep.det_a is not None else None,
                "level_nodes": list(rep.level_nodes)}

    def add(tag, text, d, a, n, cfg=None, with_implr=False, **extra):
        f = exprcore.parse(text, d)
        rule = korobov_vector(a, n, d)
        counts = axis_counts(rule)
        t0 = time.perf_counter()
        value, rep = mdi_lr(f, d, a, n, cfg=cfg, with_report=True)
        secs = time.perf_counter() - t0
        rec = {"tag": tag, "text": text, "d": d, "a": a, "n": str(n),
               "counts": [str(x) for x in counts], "value": hx(value),
               "ref_seconds": secs, **rep_fields(rep), **extra}
        if cfg is not None:
            rec["direct_cap"] = cfg.direct_cap
        if with_implr:
            rec["implr"] = hx(implr_integrate(f, d, a, n).value)
            rec["direct_sum"] = hx(direct_tensor_sum(f, midpoint_grids(rule)))
        out.append(rec)
        return rec

    # acceptance-01 sweep (reference tests/test_acceptance.py:52-71)
    for entry in corpus.entries():
        for d in range(2, 7):
            if d < entry.min_d:
                continue
            for a in range(2, 6):
                add(f"acc01_{entry.id}_d{d}_a{a}", entry.text, d, a, a**d, with_implr=True,
                    corpus=entry.id)
    add("readme_gaussian_d10", corpus.get("gaussian").text, 10, 10, 1 + 10**10,
        reference=hx(corpus.reference_value("gaussian", 10)))
    add("gaussian_d12", corpus.get("gaussian").text, 12, 10, 1 + 10**12,
        reference=hx(corpus.reference_value("gaussian", 12)))
    add("expalt_d20_a8", corpus.get("expalt").text, 20, 8, 8**20)
    add("ratprod_d4_a3_n81", corpus.get("ratprod").text, 4, 3, 81, with_implr=True)
    add("gaussian_d4_a3_n81", corpus.get("gaussian").text, 4, 3, 81, with_implr=True)
    add("expalt_d5_a2_n32", corpus.get("expalt").text, 5, 2, 32, with_implr=True)
    add("const1_d2", "1", 2, 10, 101)
    add("gaussian_d3_a7_n400", corpus.get("gaussian").text, 3, 7, 400, with_implr=True)
    add("expsum_d3_a100", corpus.get("expsum").text, 3, 100, 10**6 + 1, with_implr=True)
    add("expxy_d2_a200", corpus.get("expxy").text, 2, 200, 40001, with_implr=True)
    add("cos_lin_small_d8", "cos(0.3 + sum(i=1..d, 0.2*i*x[i]))", 8, 4, 4**8, with_implr=True)
    add("ratprod_d30_a16", corpus.get("ratprod").text, 30, 16, 16**30)
    add("gaussian_d100_a8", corpus.get("gaussian").text, 100, 8, 8**100)

    cfg2 = make_config(2)
    add("cfg2", cfg2.text, cfg2.d, cfg2.mdi_a, cfg2.mdi_n)
    cfg1 = make_config(1)
    if not skip_slow:
        add("cfg1", cfg1.text, cfg1.d, cfg1.mdi_a, cfg1.mdi_n,
            cfg=MdiConfig(direct_cap=10**10))
    # the default cap refuses config 1 (a^3 > 1e8): record the refusal too
    try:
        mdi_lr(exprcore.parse(cfg1.text, cfg1.d), cfg1.d, cfg1.mdi_a, cfg1.mdi_n)
        refused = False
    except Exception as exc:  # GridCapError
        refused = type(exc).__name__
    out.append({"tag": "cfg1_default_cap", "refused": refused})
    if not skip_slow:
        cfg4 = make_config(4)
        rec = add("cfg4", cfg4.text, cfg4.d, cfg4.mdi_a, cfg4.mdi_n)
        rec["log_raw"] = hx(math.log(float.fromhex(rec["raw"])))
    return out


def quality_cases():
    """Lattice quality measures and constructions (lattice.py:140-311),
    SURVEY.md §8(f) item 3."""
    import warnings
    out = []

    def rule_rec(rule):
        return {"n": str(rule.n), "z": [str(c) for c in rule.z]}

    rules = [LatticeRule(5, (1,)), LatticeRule(8, (1, 3)), LatticeRule(13, (1, 5)), LatticeRule(4, (1, 2)),
             korobov_vector(7, 81, 3), korobov_vector(76, 1009, 6), korobov_vector(1234, 10007, 8),
             korobov_vector(29, 4099, 12), korobov_vector(3, 2**20 + 7, 5), LatticeRule(8191, (1, 4000, 77, 5))]
    for rule in rules:
        for alpha in (2, 4):
            with warnings.catch_warnings(record=True) as w:
                warnings.simplefilter("always")
                v = p_alpha(rule, alpha)
            out.append({"tag": f"p_alpha{alpha}", **rule_rec(rule), "alpha": alpha, "value": hx(v),
                        "warned": bool(w)})
        for wm in (None, WeightModel.anchored([1.0 / (j + 1) for j in range(rule.d)], 0.7),
                   WeightModel.unanchored([0.9 ** j for j in range(rule.d)])):
            v = shift_avg_wce_sq(rule, wm)
            out.append({"tag": "wce", **rule_rec(rule), "value": hx(v),
                        "gamma": None if wm is None else [hx(g) for g in wm.gamma],
                        "beta": None if wm is None else hx(wm.beta)})
    for n, d in ((8, 3), (13, 3), (101, 5), (257, 6), (1009, 4), (4001, 3)):
        t0 = time.perf_counter()
        z = cbc_construct(n, d).z
        out.append({"tag": "cbc", "n": n, "d": d, "z": list(z), "ref_seconds": time.perf_counter() - t0})
        wm = WeightModel.anchored([0.5 ** j for j in range(d)], 1.0)
        z = cbc_construct(n, d, wm).z
        out.append({"tag": "cbc_anchored", "n": n, "d": d, "z": list(z),
                    "gamma": [hx(g) for g in wm.gamma], "beta": hx(wm.beta)})
    for n, d, crit in ((13, 3, "wce"), (101, 4, "wce"), (101, 4, "p2"), (1009, 6, "wce"), (1009, 6, "p2"),
                       (2003, 8, "wce")):
        t0 = time.perf_counter()
        r = korobov_search(n, d, criterion=crit)
        out.append({"tag": "korobov_search", "n": n, "d": d, "criterion": crit, "a": r.z[1] if d > 1 else 1,
                    "ref_seconds": time.perf_counter() - t0})
    return out


def mc_cases():
    """quad.mc_integrate (quad.py:79-93): numpy default_rng(seed) streams; the
    first rows of the stream are frozen too, so the device generator is pinned
    point by point, not only through the mean."""
    out = []

    def add(tag, text, d, n, seed):
        f = exprcore.parse(text, d)
        r = mc_integrate(f, d, n, seed=seed)
        first = np.random.default_rng(seed).random((min(n, 64), d))
        out.append({"tag": tag, "text": text, "d": d, "n": n, "seed": seed, "value": hx(r.value),
                    "first_rows": b64(first), "first_shape": list(first.shape)})

    add("expxy_101_s0", corpus.get("expxy").text, 2, 101, 0)
    add("expxy_40001_s7", corpus.get("expxy").text, 2, 40001, 7)
    add("sinsq_10001_s1", corpus.get("sinsq").text, 2, 10001, 1)
    add("gaussian5_70000_s3", corpus.get("gaussian").text, 5, 70000, 3)
    add("ratprod7_600000_s11", corpus.get("ratprod").text, 7, 600000, 11)   # > one 2^19-row block
    add("const_2p5", "2.5", 3, 1000, 0)
    return out


def suite_cases():
    """Rows of the reference's benchmark suites (bench.py:104-211) that run in
    seconds here: test1, test2, test3, test5 (values, reference values, status)."""
    from latquad import bench as rbench
    out = []
    for suite in ("test1", "test2", "test3", "test5"):
        for spec in rbench.suite_specs(suite):
            rec = rbench._run_row(spec, 0, False)
            out.append({"suite": suite, "method": rec.method, "integrand": rec.integrand, "d": rec.d,
                        "n": str(rec.n), "a": rec.a, "status": rec.status,
                        "value": None if rec.value is None else hx(rec.value),
                        "reference": None if rec.reference is None else hx(rec.reference)})
    return out


def linform_cases(skip_slow):
    """MDI-LR of integrands that are functions of one linear form (not
    separable): the reference's level loop collapses them by like-term
    collection (exprcore.py:139-169, 390-402; mdi.py:152-165).  Suite test7's
    invpow rows (bench.py:140-143, n = 1 + 8^d, a = 8) plus a few forms with
    mixed integer coefficients; value, report fields and wall time."""
    out = []

    def add(tag, text, d, a, n, slow=False):
        if slow and skip_slow:
            return
        f = exprcore.parse(text, d)
        t0 = time.perf_counter()
        value, rep = mdi_lr(f, d, a, n, with_report=True)
        secs = time.perf_counter() - t0
        out.append({"tag": tag, "text": text, "d": d, "a": a, "n": str(n), "value": hx(value),
                    "raw": hx(rep.value), "levels": rep.levels, "base_dim": rep.base_dim,
                    "fallback": rep.fallback, "level_nodes": list(rep.level_nodes), "ref_seconds": secs})
        print(f"linform {tag}: {secs:.1f}s fallback={rep.fallback}", flush=True)

    inv = corpus.get("invpow").text
    for d in (4, 6, 8):
        add(f"invpow_d{d}", inv, d, 8, 1 + 8**d)
    add("invpow_d10", inv, 10, 8, 1 + 8**10, slow=True)
    add("recip_mixed_d4", "1/(1 + x[1] + 2*x[2] + 3*x[3] + x[4])", 4, 5, 5**4)
    add("recip_mixed_d5_a4", "1/(1 + x[1] + 2*x[2] - x[3] + x[4] + 2*x[5])^2", 5, 4, 4**5 + 3)
    add("altpow_d6", "(3 + sum(i=1..d, (-1)^i*x[i]))^(-3)", 6, 3, 3**6)
    add("sin_recip_d5", "sin(1/(1 + sum(i=1..d, x[i])))", 5, 4, 4**5)
    add("mixed_outer_d6", "1/(1 + sum(i=1..d, x[i])) + exp(-(sum(i=1..d, x[i])/d)^2)", 6, 4, 4**6)
    return out


def _fft_case_sum(case):
    """Worker: the reference's own sum of one FFT-test case: slr_integrate on
    the parsed text, or -- for |.|, which the reference grammar lacks --
    points_block + the numpy restatement exp(-|x c - c.w|)."""
    key, text, params, n, a = case
    d = text.count("x[")
    print(f"fft case {key} start", flush=True)
    rule = korobov_vector(a, n, d)
    t0 = time.perf_counter()
    # the reference's own points_block and eval_array (or, for |.|, which its
    # grammar lacks, numpy) on blocks of 2^14 rows -- slr_integrate's
    # 2^19-row blocks need ~9 GB per process at d = 2048
    rows = 1 << 14
    acc = 0.0
    if params is None:
        f = exprcore.parse(text, d)
        for start in range(0, n, rows):
            pts = points_block(rule, start, min(start + rows, n))
            vals = exprcore.eval_array(f, {i + 1: pts[:, i] for i in range(d)})
            acc += float(np.sum(vals))
            # eval_array's memo lives in a self-referencing closure: a cycle
            # that holds every intermediate column until the collector runs
            del vals
            gc.collect()
        kind = "reference"
    else:
        c = np.asarray(params["c"])
        cw = float(np.dot(c, np.asarray(params["w"])))
        for start in range(0, n, rows):
            pts = points_block(rule, start, min(start + rows, n))
            acc += float(np.sum(np.exp(-np.abs(pts @ c - cw))))
        kind = "ref_points+numpy"
    value = acc / n
    return {"key": key, "n": n, "a": a, "d": d, "kind": kind, "value": hx(value),
            "ref_seconds": time.perf_counter() - t0}


def fft_cases_job(procs, only_new=False):
    """Reference sums of every case of tests/test_gpu_fft.py (cases from
    tests/fft_cases.py), so that the FFT-form kernel meets the reference and
    not only the direct orbit kernel."""
    import multiprocessing as mp
    sys.path.insert(0, os.path.dirname(HERE))
    import fft_cases
    cases = fft_cases.all_cases()
    if only_new:
        have = set()
        path = os.path.join(HERE, "fft.json")
        if os.path.exists(path):
            with open(path) as fh:
                old = json.load(fh)["cases"]
            have = {c["key"] for c in old}
        cases = [c for c in cases if c[0] not in have]
    with mp.Pool(procs, maxtasksperchild=1) as pool:
        out = list(pool.imap(_fft_case_sum, cases, chunksize=1))
    if only_new:
        out = old + out if have else out
    return out


_PARSER_FIXED = [
    "x[1]+x[2]*3", "-x[1]^2", "x[1]^2^2", "x[1]^-2", "2/x[1]", "x[1]/4", "x[1]/x[2]", "sum(i=1..d, x[i]^i)",
    "prod(i=1..d, 1/(1+x[i]))", "sum(i=3..1, garbage + )", "sum(i=1..2, x[i], 2)", "x[1]^(1+1)*3", "x[1]^2*3",
    "exp(-x[1])*sin(pi*x[2])", "--x[1]", "1..2", "1.5e3*x[1]", "2e*x[1]", "x[3]", "x[0]", "x[1.0]",
    "sum(i=1..d, sum(j=i..d, x[i]*x[j]))", "sum(d=1..2, 1)", "x[1]^(d-1)", "x[d/2]", "x[3/2]", "x[1]^(0-2)",
    "x[1]^((-2))", "x[1]^2^-1", "cos(2*pi + sum(i=1..d, 2*x[i]))", "(x[1]", "x[1] x[2]", "e^2*x[1]", "pi",
    "3 - -x[1]", "x[1]^-(2)", "sum(i=1..2, x[i]", "sum(i=1..2, x[k])", "sum(i=2..1, x[k])", "sum(i=1..2, x[(i)])",
    "1/0", "x[1]/0.0", "x[1] @ 2", ".5*x[1]", "1.2.3", "x[2^2]", "x[-1+2]", "prod(i=1..0, x[1])", "x[1]*-x[2]",
    "(1 + sum(i=1..d, x[i]))^(-(d+1))", "abs(x[1])", "sum(i=1..3, 0.1*i*x[1])", "1/(1+x[1])/2",
    "2/(1+x[1])*3/(x[1]+2)", "x[1]^0", "(x[1]+1)^1", "exp(x[1])^3", "sum(i=1..2, sum(i=1..2, x[i]))",
    "x[1]^2^3^1", "2^-1*x[1]", "x[1]^ 2 * x[1] ^ 3", "sum(i=1..d, (-1)^(i+1)*x[i]^2)", "x[1]^(2^2)",
    "sum(i=1..4/2, x[i])", "sum(i=1..d, x[i])/d", "prod(i=1..d, (x[i]-0.5)^2 + 0.1)", "sin(x[1])^-1",
    "1e-3 + x[1]", "1E+2*x[2]", "x[1] +", "*x[1]", "sum(i=1..2 x[i])", "sum(1=1..2, x[1])", "sum(x=1..2, 1)",
    "exp x[1]", "x[1]^x[2]", "x[1]^2.0", "x[2^-1]", "x[(1)]^(2)^2", "cos()", "sum(i=1..2, )",
]


def _fuzz_texts(rng, count):
    """Random well- and ill-formed texts from a small generator of the grammar
    (numbers, x[...] with index arithmetic, + - * / ^, exp/sin/cos, sum/prod)."""
    def index(depth, names):
        r = rng.random()
        if depth > 1 or r < 0.4:
            return rng.choice([str(rng.randint(1, 3)), "d"] + list(names))
        op = rng.choice(["+", "-", "*", "/"])
        return f"({index(depth + 1, names)}{op}{index(depth + 1, names)})"

    def real(depth, names):
        r = rng.random()
        if depth > 3 or r < 0.25:
            return rng.choice([f"x[{index(1, names)}]", repr(round(rng.uniform(-3, 3), 3)), "pi", "e", "d"]
                              + list(names))
        if r < 0.55:
            return f"{real(depth + 1, names)} {rng.choice(['+', '-', '*', '/'])} {real(depth + 1, names)}"
        if r < 0.65:
            return f"({real(depth + 1, names)})^{rng.choice(['2', '-1', '(1+1)', '3', '-(2)', 'd'])}"
        if r < 0.8:
            return f"{rng.choice(['exp', 'sin', 'cos'])}({real(depth + 1, names)})"
        if r < 0.9:
            v = rng.choice(["i", "j", "k"])
            return (f"{rng.choice(['sum', 'prod'])}({v}={rng.randint(0, 2)}..{rng.choice(['d', '2', '1'])}, "
                    f"{real(depth + 1, names | {v})})")
        return f"-{real(depth + 1, names)}"

    out = []
    for _ in range(count):
        t = real(0, frozenset())
        if rng.random() < 0.3:    # mutate: drop or duplicate a character
            k = rng.randrange(len(t))
            t = t[:k] + t[k + 1:] if rng.random() < 0.5 else t[:k] + t[k] + t[k:]
        out.append(t)
    return out


def parser_cases():
    """The reference grammar (exprcore.parse, exprcore.py:486-766) on fixed and
    fuzzed texts: accepted texts with the reference's value (exprcore.eval) at
    three seeded points, rejected texts with the exception type -- the
    behaviour the product parser must reproduce (the parser must
    be the builder's own code, pinned by a golden corpus)."""
    import random
    rng = random.Random(2404)
    texts = [(t, 3) for t in _PARSER_FIXED] + [(t, 4) for t in _fuzz_texts(rng, 400)]
    texts += [(e.text, max(3, e.min_d)) for e in corpus.entries()]
    out = []
    for text, d in texts:
        rec = {"text": text, "d": d}
        try:
            f = exprcore.parse(text, d)
        except Exception as exc:
            rec["error"] = type(exc).__name__
            out.append(rec)
            continue
        pts, vals = [], []
        for _ in range(3):
            pt = {j: rng.random() for j in range(1, d + 1)}
            try:
                v = hx(exprcore.eval(f, pt))
            except Exception as exc:      # e.g. ZeroDivisionError at the point
                v = type(exc).__name__
            pts.append([hx(pt[j]) for j in range(1, d + 1)])
            vals.append(v)
        rec["points"], rec["values"] = pts, vals
        out.append(rec)
    return out


def _family_texts(rng):
    """Random members of the closed families the plain-sum kernels recognise
    (linear-form exp / cos / sin / integer powers, diagonal quadratics, shifted
    quadratic products), written in the reference grammar."""
    out = []
    for d in (3, 8, 20, 40):
        for kind in ("exp", "cos", "sin", "pow", "quad", "prodq"):
            c = [round(rng.uniform(-1.5, 1.5) / max(1.0, d / 8), 6) for _ in range(d)]
            lin = " + ".join(f"{cj!r}*x[{j + 1}]" for j, cj in enumerate(c))
            a0 = round(rng.uniform(-1, 1), 4)
            if kind == "exp":
                t = f"exp({a0!r} + {lin})"
            elif kind in ("cos", "sin"):
                t = f"{round(rng.uniform(0.5, 2), 3)!r}*{kind}({a0!r} + {lin})"
            elif kind == "pow":
                k = rng.choice([-3, -2, -1, 2, 3])
                t = f"(2.5 + {lin})^({k})"
            elif kind == "quad":
                q = " + ".join(f"{round(rng.uniform(-1, 0.3) / max(1.0, d / 8), 6)!r}*x[{j + 1}]^2" for j in range(d))
                t = f"exp({lin} + {q})"
            else:
                t = "prod(i=1..d, 1/(0.8 + (x[i] - 0.4)^2))" if d <= 8 else \
                    " * ".join(f"(({round(rng.uniform(0.5, 2), 3)!r} + (x[{j + 1}] - {round(rng.uniform(0, 1), 3)!r})^2)^(-1))"
                               for j in range(min(d, 12)))
            out.append((t, d))
    return out


def slr_fuzz_cases():
    """slr_integrate of the reference (quad.py:96-104) for every accepted text
    of the parser corpus (parser.json) and for random members of the closed
    families, on Korobov rules over primes (the orbit and FFT-form layouts),
    over n = 2^12 (lattice-sequence levels) and a composite n, and on a random
    non-Korobov z: the GPU's family recognition, bytecode and kernels against
    the reference's full sums.  `scale` = mean |f| over the same points (the
    abs tolerance for sums that cancel)."""
    import random
    rng = random.Random(8867)
    with open(os.path.join(HERE, "parser.json")) as fh:
        parsed = [c for c in json.load(fh)["cases"] if "error" not in c]
    texts = [(c["text"], c["d"]) for c in parsed] + _family_texts(rng)
    out = []
    for i, (text, d) in enumerate(texts):
        try:
            f = exprcore.parse(text, d)
        except Exception:
            continue
        if not exprcore.free_vars(f):
            continue
        lats = [("korobov", 4099 if d <= 8 else 10007), ("korobov", 4096), ("korobov", 3003), ("random", 2039)]
        for kind, n in lats[i % 2: i % 2 + 3]:
            if kind == "korobov":
                a = rng.randrange(2, n)
                while math.gcd(a, n) != 1:
                    a = rng.randrange(2, n)
                rule = korobov_vector(a, n, d)
            else:
                rule = LatticeRule(n, tuple([1] + [rng.randrange(1, n) for _ in range(d - 1)]))
            with np.errstate(all="ignore"):
                try:
                    val = slr_integrate(f, rule).value
                except Exception:
                    continue
                pts = points_block(rule, 0, n)
                vals = exprcore.eval_array(f, {j + 1: pts[:, j] for j in range(d)})
                scale = float(np.mean(np.abs(vals))) if np.ndim(vals) else abs(float(vals))
            if not (math.isfinite(val) and math.isfinite(scale)):
                continue
            out.append({"text": text, "d": d, "n": n, "z": [str(v) for v in rule.z], "kind": kind,
                        "value": hx(val), "scale": hx(scale)})
    # the closed families on prime n >= 2^18, where the orbit (direct) and
    # FFT-form (d >= 49 at n >= 2^22) layouts take the full lattice
    for (text, d), n in zip(_family_texts_big(rng), _BIG_N * 100):
        a = rng.randrange(2, n)
        rule = korobov_vector(a, n, d)
        f = exprcore.parse(text, d)
        val = slr_integrate(f, rule).value
        acc = 0.0
        for start in range(0, n, 1 << 18):
            pts = points_block(rule, start, min(n, start + (1 << 18)))
            acc += float(np.sum(np.abs(exprcore.eval_array(f, {j + 1: pts[:, j] for j in range(d)}))))
        out.append({"text": text, "d": d, "n": n, "z": [str(v) for v in rule.z], "kind": "korobov_big",
                    "value": hx(val), "scale": hx(acc / n)})
    return out


def mdi_fuzz_cases():
    """mdi_lr of the reference (mdi.py:215-234) for every accepted text of the
    parser corpus with coordinates, on Korobov grids N^d (+1) with N = 3, 4 and
    d = the text's own 3/4 and 6 (two levels): value, report fields, or the
    exception type.  `scale` = mean |f| over the midpoint grid (numpy)."""
    import itertools
    with open(os.path.join(HERE, "parser.json")) as fh:
        parsed = [c for c in json.load(fh)["cases"] if "error" not in c]
    # integrands with a factor spanning more than three axes (no separation,
    # no single linear form: the direct-sweep branch here)
    parsed = parsed + [{"text": t, "d": 4} for t in (
        "exp(x[1]*x[2]*x[3]*x[4])", "1/(1 + x[1]*x[2]*x[3]*x[4])", "sin(x[1]*x[2]*x[3] + x[4])*x[2]",
        "exp(-(x[1] - x[2])^2 - (x[3] - x[4])^2 - x[1]*x[4])", "(1 + x[1]*x[2] + x[3]*x[4])^(-2)",
        "cos(x[1] + x[2]*x[3]*x[4]) + exp(x[1]*x[2]*x[3]*x[4])")]
    out = []
    for i, c in enumerate(parsed):
        text = c["text"]
        for d, a, extra in ((c["d"], 3 + i % 2, 1), (6, 3, i % 2)):
            n = a ** d + extra
            try:
                f = exprcore.parse(text, d)
            except Exception:
                continue
            if not exprcore.free_vars(f):
                continue
            rec = {"text": text, "d": d, "a": a, "n": n}
            t0 = time.perf_counter()
            try:
                with np.errstate(all="ignore"):
                    val, rep = mdi_lr(f, d, a, n, with_report=True)
                rec.update(value=hx(val), levels=rep.levels, base_dim=rep.base_dim, fallback=rep.fallback)
                counts = axis_counts(korobov_vector(a, n, d))
                grid = [(np.arange(k) + 0.5) / k for k in counts]
                mesh = np.meshgrid(*grid, indexing="ij")
                with np.errstate(all="ignore"):
                    vals = exprcore.eval_array(f, {j + 1: mesh[j].reshape(-1) for j in range(d)})
                rec["scale"] = hx(float(np.mean(np.abs(vals))) if np.ndim(vals) else abs(float(vals)))
            except Exception as exc:
                rec["error"] = type(exc).__name__
            rec["ref_seconds"] = round(time.perf_counter() - t0, 4)
            if "value" in rec and not (math.isfinite(float.fromhex(rec["value"])) and
                                       math.isfinite(float.fromhex(rec["scale"]))):
                continue
            out.append(rec)
    # past the direct cap, where the reference's levels still fit the node
    # budget: it sweeps only its base axes (no GridCapError)
    for text, d, a in (("exp(x[1]*x[2]*x[3]*x[4]*x[5])", 5, 45),
                       ("exp(-(x[1] - x[2])^2 - (x[3] - x[4])^2 - x[1]*x[4] - x[5])", 5, 42)):
        f = exprcore.parse(text, d)
        t0 = time.perf_counter()
        val, rep = mdi_lr(f, d, a, a ** d, with_report=True)
        out.append({"text": text, "d": d, "a": a, "n": a ** d, "value": hx(val), "levels": rep.levels,
                    "base_dim": rep.base_dim, "fallback": rep.fallback, "scale": hx(abs(val)),
                    "ref_seconds": round(time.perf_counter() - t0, 4), "over_cap": True})
    return out


def linform_w_cases():
    """mdi_lr of the reference for products of separable real weights and a
    function of one commensurate linear form (its like-term collection carries
    node-dependent coefficients, exprcore.py:139-206): value and report,
    including grids past the direct cap (d = 10, 12) and weights on axes the
    linear form does not use."""
    cases = [("exp(-sum(i=1..d, x[i]^2))*(1 + sum(i=1..d, x[i]))^(-2)", 6, 8, 8**6 + 1),
             ("exp(-sum(i=1..d, x[i]^2))*(1 + sum(i=1..d, x[i]))^(-2)", 10, 8, 8**10 + 1),
             ("exp(-sum(i=1..d, x[i]^2))*(1 + sum(i=1..d, x[i]))^(-2)", 12, 8, 8**12 + 1),
             ("x[1]*x[2]*(1 + sum(i=1..d, x[i]))^(-3)", 5, 4, 4**5 + 1),
             ("prod(i=1..d, 1 + x[i])*exp(-(sum(i=1..d, x[i]))^2)", 7, 6, 6**7 + 1),
             ("prod(i=1..d, 1 + x[i])*exp(-((sum(i=1..d, x[i]))^2))", 9, 6, 6**9 + 1),
             ("x[5]^2*(1 + x[1] + x[2] + x[3])^(-2)", 5, 5, 5**5 + 1),
             ("exp(-sum(i=1..d, x[i]^2))*(3 + x[1] - x[2] + x[3] - 0.5*x[4])^(-1)", 6, 8, 8**6),
             ("(x[1] - 0.5)*cos(x[2])*(2 + x[1] + 2*x[2] + x[3])^(-2)", 4, 6, 6**4 + 1),
             # sums whose terms collapse by different branches
             ("(1 + sum(i=1..d, x[i]))^(-2) + exp(-sum(i=1..d, x[i]^2))", 10, 8, 8**10 + 1),
             ("3*(2 + sum(i=1..d, x[i]))^(-1) - 0.5*prod(i=1..d, 1 + x[i]) + 1.25", 8, 8, 8**8 + 1),
             ("x[1]*x[2]*(1 + sum(i=1..d, x[i]))^(-3) + cos(sum(i=1..d, x[i]))", 9, 6, 6**9 + 1),
             # functions of two commensurate linear forms
             ("(1 + sum(i=1..d, x[i]))^(-2)*(2 + sum(i=1..d, (-1)^i*x[i]))^(-1)", 8, 8, 8**8 + 1),
             ("(1 + sum(i=1..d, x[i]))^(-2)*(2 + sum(i=1..d, (-1)^i*x[i]))^(-1)", 10, 8, 8**10 + 1),
             ("exp(-((sum(i=1..d, x[i]) - 0.5*d)^2)/d)*cos(sum(i=1..d, i*x[i])/d)", 8, 6, 6**8 + 1),
             ("1/(1 + (x[1] + x[2] + x[3] - x[4])^2 + (x[1] - 2*x[2] + 0.5*x[5])^2)", 6, 5, 5**6 + 1)]
    out = []
    for text, d, a, n in cases:
        f = exprcore.parse(text, d)
        t0 = time.perf_counter()
        val, rep = mdi_lr(f, d, a, n, with_report=True)
        out.append({"text": text, "d": d, "a": a, "n": n, "value": hx(val), "levels": rep.levels,
                    "base_dim": rep.base_dim, "fallback": rep.fallback,
                    "ref_seconds": round(time.perf_counter() - t0, 3)})
    # the level-plan options (m axes per level, stripping order) on the same branches
    for text, d, a, n in cases[:1] + cases[3:5] + cases[9:10] + cases[12:13]:
        for m, order in ((2, "forward"), (1, "reverse"), (3, "reverse")):
            f = exprcore.parse(text, d)
            cfg = MdiConfig(m=m, order=order)
            val, rep = mdi_lr(f, d, a, n, cfg=cfg, with_report=True)
            out.append({"text": text, "d": d, "a": a, "n": n, "m": m, "order": order, "value": hx(val),
                        "levels": rep.levels, "base_dim": rep.base_dim, "fallback": rep.fallback})
    return out


_BIG_N = [262147, 1048583, 4194319]


def _family_texts_big(rng):
    out = []
    for d in (8, 40, 64, 100):
        for kind in ("exp", "cos", "sin", "pow", "quad"):
            c = [round(rng.uniform(0.0, 1.0) * 3.0 / d, 6) for _ in range(d)]
            lin = " + ".join(f"{cj!r}*x[{j + 1}]" for j, cj in enumerate(c))
            if kind == "exp":
                t = f"exp(-0.5 + {lin})"
            elif kind in ("cos", "sin"):
                t = f"{kind}(0.25 + {lin})"
            elif kind == "pow":
                t = f"(1.5 + {lin})^(-2)"
            else:
                q = " + ".join(f"{round(-rng.uniform(0.0, 1.0) * 3.0 / d, 6)!r}*x[{j + 1}]^2" for j in range(d))
                t = f"exp({lin} + {q})"
            out.append((t, d))
    return out


def suite7_cases():
    """Suite test7 (bench.py:140-143: MDI-LR over d at n = 8^d + 1, a = 8) rows
    with d <= 10 from the reference's own row runner: expalt, ratprod,
    gaussian, coslin, expsq (separable) and invpow (collapses by like-term
    collection; d = 10 takes ~7 min here)."""
    from latquad import bench as rbench
    out = []
    for spec in rbench.suite_specs("test7"):
        if spec[2] > 10:
            continue
        t0 = time.perf_counter()
        rec = rbench._run_row(spec, 0, False)
        out.append({"suite": "test7", "method": rec.method, "integrand": rec.integrand, "d": rec.d,
                    "n": str(rec.n), "a": rec.a, "status": rec.status,
                    "value": None if rec.value is None else hx(rec.value),
                    "reference": None if rec.reference is None else hx(rec.reference),
                    "ref_seconds": time.perf_counter() - t0})
        print(f"suite7 {spec}: {time.perf_counter() - t0:.1f}s", flush=True)
    return out


def subgrid_cases():
    """MDI-LR of integrands that are not separable axis by axis: pieces on a
    few axes (cores) times separable factors, and integrands that leave axes
    unused.  The reference's levels strip the separable and unused axes and
    sweep the rest (mdi.py:152-183)."""
    out = []
    for tag, text, d, a, n in (("expxy_d10", "exp(x[1]*x[2])", 10, 8, 8**10 + 1),
                               ("corpus_expxy_d6", corpus.get("expxy").text, 6, 5, 5**6),
                               ("recip3_d8", "1/(1 + x[1]*x[2] + x[3])", 8, 6, 6**8 + 7),
                               ("exp_x1x9_d10", "exp(x[1]*x[9])", 10, 4, 4**10),
                               ("exp4_d8", "exp(x[1]*x[2]*x[3]*x[4])", 8, 4, 4**8),
                               ("core_times_prod_d8", "exp(x[1]*x[2])*prod(i=3..d, 1/(1 + x[i]^2))", 8, 6, 6**8),
                               ("core_phasor_d7", "cos(x[1]*x[7] + x[2]) + x[3]*x[4]*x[5]", 7, 5, 5**7),
                               ("recip_core_d9", "(1 + x[1] + x[2] + x[3])^(-3)*exp(sum(i=4..d, x[i])/d)",
                                9, 4, 4**9 + 1)):
        f = exprcore.parse(text, d)
        t0 = time.perf_counter()
        value, rep = mdi_lr(f, d, a, n, with_report=True)
        out.append({"tag": tag, "text": text, "d": d, "a": a, "n": str(n), "value": hx(value),
                    "raw": hx(rep.value), "levels": rep.levels, "base_dim": rep.base_dim,
                    "fallback": rep.fallback, "ref_seconds": time.perf_counter() - t0})
    return out


def _cfg5_chunk(args):
    """Worker: the reference's own points_block (lattice.py:96-105) over
    [lo, hi) in blocks of 2^15 rows, integrand exp(-|x @ c - c.w|) in numpy
    (the reference grammar has no abs, exprcore.py:638).  Returns the block
    sums (np.sum, pairwise) in index order."""
    lo, hi = args
    cfg = make_config(5)
    rule = LatticeRule(cfg.plain_n, cfg.plain_z())
    c = np.asarray(cfg.c)
    cw = float(np.dot(c, np.asarray(cfg.w)))
    sums = []
    blk = 1 << 15
    for s in range(lo, hi, blk):
        pts = points_block(rule, s, min(s + blk, hi))
        sums.append(float(np.sum(np.exp(-np.abs(pts @ c - cw)))))
    return sums


def cfg5_full_case(procs):
    """Config 5's plain sum over ALL n = 2^31 - 1 points from the reference's
    own points_block.  Contiguous index chunks
    of 2^22 points in `procs` processes; the block sums are combined with
    math.fsum (correctly rounded), so the frozen total does not depend on the
    process count.  About 70 min on 8 cores."""
    import multiprocessing as mp
    cfg = make_config(5)
    n = cfg.plain_n
    step = 1 << 22
    chunks = [(lo, min(lo + step, n)) for lo in range(0, n, step)]
    t0 = time.perf_counter()
    block_sums = []
    with mp.Pool(procs) as pool:
        for k, sums in enumerate(pool.imap(_cfg5_chunk, chunks)):
            block_sums.extend(sums)
            if k % 32 == 0:
                print(f"cfg5_full: chunk {k}/{len(chunks)} {time.perf_counter() - t0:.0f}s", flush=True)
    total = math.fsum(block_sums)
    return [{"tag": "cfg5_full", "kind": "ref_points+numpy", "text": cfg.text, "d": cfg.d,
             "n": str(n), "a": cfg.plain_a, "i_begin": 0, "i_end": n, "block_rows": 1 << 15,
             "n_blocks": len(block_sums), "sum_fsum": hx(total), "value": hx(total / n),
             "procs": procs, "ref_seconds": time.perf_counter() - t0}]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--skip-slow", action="store_true")
    ap.add_argument("--only", choices=["points", "slr", "mdi", "quality", "mc", "suites", "cfg5_full", "linform", "fft", "parser", "suites7", "subgrid", "slr_fuzz", "mdi_fuzz", "linform_w"],
                    default=None)
    ap.add_argument("--procs", type=int, default=os.cpu_count())
    ap.add_argument("--only-new", action="store_true", help="fft: compute only cases missing from fft.json")
    args = ap.parse_args()
    meta = {"generator": "tests/golden/make_golden.py", "numpy": np.__version__,
            "python": sys.version.split()[0], "reference": "/root/reference/pkg (latquad 0.1.0)"}
    jobs = {"points": lambda: points_cases(), "slr": lambda: slr_cases(args.skip_slow),
            "mdi": lambda: mdi_cases(args.skip_slow), "quality": quality_cases, "mc": mc_cases,
            "suites": suite_cases, "cfg5_full": lambda: cfg5_full_case(args.procs),
            "linform": lambda: linform_cases(args.skip_slow), "fft": lambda: fft_cases_job(args.procs, args.only_new),
            "parser": parser_cases, "suites7": suite7_cases, "subgrid": subgrid_cases,
            "slr_fuzz": slr_fuzz_cases, "mdi_fuzz": mdi_fuzz_cases, "linform_w": linform_w_cases}
    for name, fn in jobs.items():
        if args.only != name and (args.only or name in ("cfg5_full", "linform", "fft", "suites7", "slr_fuzz", "mdi_fuzz", "linform_w")):
            continue
        t0 = time.perf_counter()
        cases = fn()
        with open(os.path.join(HERE, f"{name}.json"), "w") as fh:
            json.dump({"meta": meta, "cases": cases}, fh, indent=1)
        print(f"{name}: {len(cases)} cases in {time.perf_counter() - t0:.1f}s", flush=True)


if __name__ == "__main__":
    main()
