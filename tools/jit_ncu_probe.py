"""One JIT lattice-kernel case for ncu (the paper's test3 Gaussian SLR row at
d = 10, n = 10^10 + 1, stepped 64-bit residues): a warm call, then timed calls.

    python tools/jit_ncu_probe.py [d]           (GPU box)
    ncu --set full -k regex:lq_jit_lattice -s 1 -c 1 python tools/jit_ncu_probe.py
"""

import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import paper_2404_08867_b200 as lq

    d = int(sys.argv[1]) if len(sys.argv) > 1 else 10
    a = {10: 76069, 11: 35963, 12: 47987}[d]
    f = lq.parse("0.3989422804014327*exp(-sum(i=1..d, x[i]^2)/2)", d)
    rule = lq.korobov_vector(a, 10**d + 1, d)
    v = lq.slr_integrate(f, rule).value
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        v2 = lq.slr_integrate(f, rule).value
        ts.append(time.perf_counter() - t0)
    assert v2 == v
    print(f"d={d} n=10^{d}+1 value={v.hex()} best_s={min(ts):.4f}")


if __name__ == "__main__":
    main()
