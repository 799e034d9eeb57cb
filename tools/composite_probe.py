"""Composite-modulus Korobov rules: wall time of the full
plain sum through the divisor-class plan vs the mirror-paired index kernel
(LQ_ORBIT=0), config 5's integrand (d = 1000) and a d = 100 exp family."""
import math, os, random, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_08867_b200 as lq
from paper_2404_08867_b200 import _native as N, engine
from paper_2404_08867_b200.configs import make_config

def best(fn, k=3):
    fn()
    out = 1e30
    for _ in range(k):
        t = time.perf_counter(); v = fn(); out = min(out, time.perf_counter() - t)
    return out, v

cfg = make_config(5)
rng = random.Random(9)
for n in (2**31 - 2, 2**31 - 1 - 2**16 * 3, 10**9, 3 * 5 * 7 * 11 * 13 * 17 * 19 * 23 * 29):
    for text, d in ((cfg.text, cfg.d), ("exp(-0.5 + " + " + ".join(f"{0.03 * (1 + j % 7)!r}*x[{j + 1}]" for j in range(100)) + ")", 100)):
        a = rng.randrange(2, n)
        while math.gcd(a, n) != 1:
            a = rng.randrange(2, n)
        f = lq.parse(text, d)
        z = lq.korobov_vector(a, n, d).z_reduced_array()
        pi = engine.plain_integrand(f, d)
        mode = N.lattice_layout(pi.struct, n, z).mode
        t1, v1 = best(lambda: engine.lattice_sum(pi, n, z))
        os.environ["LQ_ORBIT"] = "0"
        pi0 = engine.plain_integrand(lq.parse(text, d), d)
        t0, v0 = best(lambda: engine.lattice_sum(pi0, n, z), 2)
        del os.environ["LQ_ORBIT"]
        print(f"n={n} d={d} mode={mode}: plan {t1 * 1e3:.2f} ms, paired {t0 * 1e3:.2f} ms ({t0 / t1:.1f}x), "
              f"rel diff {abs(v1 - v0) / abs(v0):.1e}", flush=True)
