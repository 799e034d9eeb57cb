"""Stepped vs per-point modular coordinates in the JIT lattice kernel
(jit.py: LQ_STEP): the paper's test3 Gaussian rows past n = 2^31 (and one
n <= 2^31 program) timed both ways through slr_integrate; the sums must be
bit-identical (same coordinates, same order).

    python tools/jit_step_probe.py            (GPU box)
"""

import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import paper_2404_08867_b200 as lq
    from paper_2404_08867_b200 import engine, jit

    gauss = "0.3989422804014327*exp(-sum(i=1..d, x[i]^2)/2)"
    cases = [(gauss, 10, 10**10 + 1, 76069), (gauss, 11, 10**11 + 1, 35963), (gauss, 12, 10**12 + 1, 47987),
             ("x[2]*exp(x[1]*x[3]) + sin(x[1]^2)", 3, 2147483647, 48271)]
    rows = []
    if "--implr-only" in sys.argv:
        cases = []
    for text, d, n, a in cases:
        f = lq.parse(text, d)
        rule = lq.korobov_vector(a, n, d)
        row = {"text": text[:40], "d": d, "n": n}
        for label, cap in (("per_point", 0), ("stepped", 24)):
            jit.STEP_MAX_VARS = cap
            jit._cache.clear()
            engine._plain_cache.clear()
            v = lq.slr_integrate(f, rule).value          # includes the NVRTC compile
            reps = 1 if n >= 10**12 else 3
            ts = []
            for _ in range(reps):
                t0 = time.perf_counter()
                v2 = lq.slr_integrate(f, rule).value
                ts.append(time.perf_counter() - t0)
            assert v2 == v
            row[label + "_s"] = min(ts)
            row[label + "_value"] = v.hex()
        row["identical"] = row["per_point_value"] == row["stepped_value"]
        row["speedup"] = row["per_point_s"] / row["stepped_s"]
        rows.append(row)
        print(json.dumps(row), flush=True)
    # direct tensor-grid sums (implr_integrate, the paper's Imp-LR rows)
    for d in (10, 11, 12):
        f = lq.parse(gauss, d)
        n = 10**d + 1
        row = {"text": "implr " + gauss[:30], "d": d, "n": n}
        for label, cap in (("per_point", 0), ("stepped", 24)):
            jit.STEP_MAX_VARS = cap
            jit._cache.clear()
            v = lq.implr_integrate(f, d, 10, n, cap=10**13).value
            t0 = time.perf_counter()
            v2 = lq.implr_integrate(f, d, 10, n, cap=10**13).value
            row[label + "_s"] = time.perf_counter() - t0
            assert v2 == v
            row[label + "_value"] = v.hex()
        row["identical"] = row["per_point_value"] == row["stepped_value"]
        row["speedup"] = row["per_point_s"] / row["stepped_s"]
        rows.append(row)
        print(json.dumps(row), flush=True)
    os.makedirs("gpurun_out", exist_ok=True)
    with open("gpurun_out/jit_step_probe.json", "w") as fh:
        json.dump(rows, fh, indent=1)


if __name__ == "__main__":
    main()
