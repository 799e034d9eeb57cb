"""Random functions of linear forms through the FFT-form chains (LQ_FFT=always)
against the oracle's literal evaluator: the closed families (exp, sin+cos,
exp-abs, integer powers, the diagonal Gaussian) and one-form programs
(LQ_FAM_LIN_PROG) with random coefficients, on full Korobov lattices over
random primes, 2^k and composite n.  Exit 1 on any mismatch above 1e-10.

    LQ_FFT=always python tools/fuzz_fft_vs_oracle.py [cases] [seed]   (GPU box)
"""
import math
import os
import random
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_08867_b200 as lq  # noqa: E402
from oracle import np_oracle  # noqa: E402
from paper_2404_08867_b200 import _native as N, engine  # noqa: E402


def is_prime(m):
    if m < 2:
        return False
    for p in range(2, int(m ** 0.5) + 1):
        if m % p == 0:
            return False
    return True


def form(rng, d, scale):
    cs = [rng.uniform(-1.0, 1.0) for _ in range(d)]
    s = sum(abs(c) for c in cs)
    cs = [scale * c / s for c in cs]
    return " + ".join(f"{c!r}*x[{j + 1}]" for j, c in enumerate(cs))


def text_for(rng, d):
    L = form(rng, d, rng.uniform(0.5, 6.0))
    kind = rng.choice(["exp", "sincos", "expabs", "pow", "gauss", "prog1", "prog2"])
    if kind == "exp":
        return f"exp({L})"
    if kind == "sincos":
        return f"0.3*sin({L}) + 1.7*cos({L})"
    if kind == "expabs":
        return f"exp(-abs({L} - {rng.uniform(-1, 1)!r}))"
    if kind == "pow":
        return f"(2.5 + {form(rng, d, 1.5)})^(-{rng.randint(1, 4)})"
    if kind == "gauss":
        return "exp(-(" + " + ".join(f"{rng.uniform(0.1, 2.0)!r}*(x[{j + 1}] - {rng.random()!r})^2"
                                     for j in range(d)) + ")/" + repr(float(d)) + ")"
    if kind == "prog1":
        return f"1/(1 + ({L})^2)"
    return f"cos({L})^2 + sin(3*({L}))"


def main():
    cases = int(sys.argv[1]) if len(sys.argv) > 1 else 60
    rng = random.Random(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
    bad = 0
    layouts = {}
    for case in range(cases):
        d = rng.choice([2, 3, 5, 8, 13, 24, 49, 64])
        shape = rng.choice(["prime", "pow2", "composite"])
        if shape == "pow2":
            n = 1 << rng.randint(14, 18)
        else:
            n = rng.randint(30000, 250000)
            while is_prime(n) != (shape == "prime"):
                n += 1
        a = rng.randrange(2, n)
        while math.gcd(a, n) != 1:
            a = rng.randrange(2, n)
        text = text_for(rng, d)
        f = lq.parse(text, d)
        rule = lq.korobov_vector(a, n, d)
        lay = N.lattice_layout(engine.plain_integrand(f, d).struct, n, rule.z_reduced_array())
        layouts[lay.mode] = layouts.get(lay.mode, 0) + 1
        got = lq.slr_integrate(f, rule).value * n
        want = np_oracle.slr_sum(text, n, rule.z)
        tol = 1e-10 * max(abs(want), 1e-3 * n)
        if not abs(got - want) <= tol:
            bad += 1
            print(f"MISMATCH case {case}: n={n} a={a} d={d} layout={lay.mode} got={got!r} want={want!r}\n  {text[:200]}",
                  flush=True)
    print(f"{cases} cases, {bad} mismatches, layouts {layouts}")
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
