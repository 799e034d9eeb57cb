"""Randomised sweep of Korobov rules over composite n: the
divisor-class layout against the mirror-paired index kernel (LQ_ORBIT=0) for
random moduli, multipliers, dimensions and families.  Prints one line per
mismatch and a summary; exit status 1 on any mismatch above 1e-12."""
import math, os, random, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_08867_b200 as lq
from paper_2404_08867_b200 import _native as N, engine

rng = random.Random(int(sys.argv[2]) if len(sys.argv) > 2 else 2024)
cases = int(sys.argv[1]) if len(sys.argv) > 1 else 200
modes, bad = {}, 0
for k in range(cases):
    while True:   # a composite modulus, not a power of two
        n = rng.choice([rng.randrange(1 << 12, 1 << 20), rng.randrange(1 << 20, 1 << 26), rng.randrange(1 << 26, 1 << 31)])
        if n & (n - 1) and any(n % p == 0 for p in range(2, int(n ** 0.5) + 1)):
            break
    a = rng.randrange(2, n)
    while math.gcd(a, n) != 1:
        a = rng.randrange(2, n)
    d = rng.choice([4, 9, 30, 60, 130, 400])
    fam = rng.choice(["exp", "expabs", "cos", "quad", "pow"])
    c = [rng.uniform(0.1, 1.0) * 3.0 / d for _ in range(d)]
    lin = " + ".join(f"{cj!r}*x[{j + 1}]" for j, cj in enumerate(c))
    text = {"exp": f"exp(-0.5 + {lin})", "expabs": f"exp(-abs({lin} - 1.1))", "cos": f"cos(0.2 + {lin})",
            "pow": f"(1.5 + {lin})^(-2)",
            "quad": "exp(" + lin + " + " + " + ".join(f"{-rng.uniform(0, 1) * 3.0 / d!r}*x[{j + 1}]^2"
                                                   for j in range(d)) + ")"}[fam]
    f = lq.parse(text, d)
    z = lq.korobov_vector(a, n, d).z_reduced_array()
    pi = engine.plain_integrand(f, d)
    mode = N.lattice_layout(pi.struct, n, z).mode
    modes[mode] = modes.get(mode, 0) + 1
    got = engine.lattice_sum(pi, n, z)
    os.environ["LQ_ORBIT"] = "0"
    ref = engine.lattice_sum(engine.plain_integrand(lq.parse(text, d), d), n, z)
    del os.environ["LQ_ORBIT"]
    if not math.isclose(got, ref, rel_tol=1e-12, abs_tol=1e-12 * n):
        bad += 1
        print(f"MISMATCH n={n} a={a} d={d} {fam} mode={mode}: {got!r} vs {ref!r}", flush=True)
print(f"{cases} cases, {bad} mismatches, layout modes {modes}")
sys.exit(1 if bad else 0)
