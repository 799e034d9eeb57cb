"""Integrand families and lattice cases of the FFT-form tests
(tests/test_gpu_fft.py), shared with tests/golden/make_golden.py, which
freezes the reference's own sums for every case (tests/golden/fft.json) so
that the FFT kernel meets a reference value, not only another GPU kernel."""

import zlib

import numpy as np

FAMILIES = ["exp", "sincos", "expabs", "pow", "gauss", "qtrig"]
MAIN = [(100003, 37, "primitive"), (100003, 200, "odd_order"),
        (1000003, 600, "even_order_cosets"), (1000003, 2048, "primitive")]
PAIR = [("expabs", 10.0, 0), ("expabs", 0.01, 0), ("expabs", 350.0, 0), ("expabs", 800.0, 0),
        ("exp", 3.0, 0.25), ("exp", 600.0, 0.25), ("exp", 100.0, -650.0), ("sincos", 9.0, 0),
        ("sincos", 400.0, 0)]
RM_FAMILIES = ["exp", "expabs", "sincos"]
# functions of one linear form no closed family covers (PlainFamily 'lin_prog':
# the FFT-form chains with the outer G run as bytecode)
LINPROG = [("recip_sq", 100003, 64), ("gauss_lin", 1000003, 300), ("trig_mix", 100003, 150),
           ("recip_sq", 100003, 700)]
RM_DS = [768, 769, 1024, 1025]
_FACTORS = {100003: (2, 3, 7, 2381), 1000003: (2, 3, 166667)}


def family_text(family, d, rng):
    """Expression text of a family with rng-drawn coefficients c, w; the
    second value is the numpy form (params) for texts the reference grammar
    cannot parse (|.|, exprcore.py:638)."""
    c = [float(v) for v in rng.uniform(0, 1, d)]
    w = [float(v) for v in rng.uniform(0, 1, d)]
    if family == "exp":
        return "exp(" + " + ".join(f"{c[j] / d!r}*x[{j + 1}]" for j in range(d)) + ")", None
    if family == "sincos":
        return "cos(0.7 + " + " + ".join(f"{c[j]!r}*x[{j + 1}]" for j in range(d)) + ")", None
    if family == "expabs":
        cc = [v / 4 for v in c]
        return ("exp(-abs(" + " + ".join(f"{cc[j]!r}*(x[{j + 1}] - {w[j]!r})" for j in range(d)) + "))",
                {"kind": "expabs", "c": cc, "w": w, "offset": 0.0})
    if family == "pow":
        return "(1.5 + " + " + ".join(f"{c[j] / d!r}*x[{j + 1}]" for j in range(d)) + ")^(-3)", None
    if family == "qtrig":
        return "0.5 + sin(0.3 + " + " + ".join(f"{c[j] ** 2 / 4!r}*(x[{j + 1}] - {w[j]!r})^2"
                                               for j in range(d)) + ")", None
    return "exp(-(" + " + ".join(f"{c[j] ** 2 / 4!r}*(x[{j + 1}] - {w[j]!r})^2" for j in range(d)) + "))", None


def pair_text(family, d, rng, scale, offset):
    c = rng.uniform(0, 1, d)
    c = c * (scale / c.sum())
    w = rng.uniform(0, 1, d)
    if family == "expabs":
        cc, ww = [float(v) for v in c], [float(v) for v in w]
        return ("exp(-abs(" + " + ".join(f"{cc[j]!r}*(x[{j + 1}] - {ww[j]!r})" for j in range(d)) + "))",
                {"kind": "expabs", "c": cc, "w": ww, "offset": 0.0})
    sgn = np.where(rng.uniform(size=d) < 0.5, -1.0, 1.0)
    if family == "exp":
        return (f"exp({offset!r} + " + " + ".join(f"{float(sgn[j] * c[j])!r}*x[{j + 1}]" for j in range(d)) + ")",
                None)
    return ("2.0 + 0.5*cos(1.3 + " + " + ".join(f"{float(sgn[j] * c[j])!r}*x[{j + 1}]" for j in range(d)) + ")",
            None)


def primitive_root(n):
    g = 2
    while any(pow(g, (n - 1) // p, n) == 1 for p in _FACTORS[n]):
        g += 1
    return g


def main_case(family, n, d, kind):
    """(key, text, params, n, a) of test_fft_matches_direct_orbit_and_oracle."""
    g = primitive_root(n)
    a = {"primitive": g, "odd_order": pow(g, 2, n), "even_order_cosets": pow(g, 3, n)}[kind]
    rng = np.random.default_rng(zlib.crc32(f"{family}/{n}/{d}".encode()))
    text, params = family_text(family, d, rng)
    return f"main/{family}/{n}/{d}/{kind}", text, params, n, a


def pair_case(family, scale, offset):
    n, d, a = 100003, 150, 2
    rng = np.random.default_rng(zlib.crc32(f"pair/{family}/{scale}".encode()))
    text, params = pair_text(family, d, rng, scale, offset)
    return f"pair/{family}/{scale}/{offset}", text, params, n, a


def rm_case(family, d):
    n = 100003
    rng = np.random.default_rng(zlib.crc32(f"rm/{family}/{d}".encode()))
    text, params = family_text(family, d, rng)
    return f"rm/{family}/{d}", text, params, n, primitive_root(n)


def linprog_text(kind, d, rng):
    c = [float(v) for v in rng.uniform(0, 1, d)]
    L = " + ".join(f"{c[j] / d!r}*x[{j + 1}]" for j in range(d))
    if kind == "recip_sq":
        return f"1/(1 + (2*({L}) - 0.8)^2)"
    if kind == "gauss_lin":
        return f"exp(-(3*({L}) - 1.5)^2)"
    return f"cos({L})^2 + 0.5*sin(3*({L}))"


def linprog_case(kind, n, d):
    rng = np.random.default_rng(zlib.crc32(f"linprog/{kind}/{n}/{d}".encode()))
    return f"linprog/{kind}/{n}/{d}", linprog_text(kind, d, rng), None, n, primitive_root(n)


def all_cases():
    out = [main_case(f, n, d, k) for f in FAMILIES for (n, d, k) in MAIN]
    out += [pair_case(*p) for p in PAIR]
    out += [rm_case(f, d) for f in RM_FAMILIES for d in RM_DS]
    out += [linprog_case(*c) for c in LINPROG]
    return out
