"""FFT-form vs direct orbit kernel over d (exp-abs linear family, Korobov
rules on prime n): where should orbit_for switch to the FFT form?"""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2404_08867_b200 as lq
from paper_2404_08867_b200 import _native as N, engine

h = N.lib(); ctx = N.ctx(); N.check(h.lq_ctx_enable_timing(ctx, 1))


def kernel_ms(pi, n, z, mode):
    os.environ["LQ_FFT"] = mode
    lay = N.lattice_layout(pi.struct, n, z).mode
    engine.lattice_sum(pi, n, z)
    best = 1e30
    for _ in range(3):
        s = engine.lattice_sum(pi, n, z)
        kms, nl = C.c_float(), C.c_int64(); N.check(h.lq_last_kernel_ms(ctx, C.byref(kms), C.byref(nl)))
        best = min(best, kms.value)
    return best, lay, s


def text_of(fam, d, rng):
    c = rng.uniform(0, 1, d); c *= 10 / c.sum(); w = rng.uniform(0, 1, d)
    if fam == "pow":
        return "(1.5 + " + " + ".join(f"{float(c[j]) / 10!r}*x[{j + 1}]" for j in range(d)) + ")^(-3)"
    if fam == "expabs":
        return "exp(-abs(" + " + ".join(f"{float(c[j])!r}*(x[{j + 1}] - {float(w[j])!r})" for j in range(d)) + "))"
    if fam == "sincos":
        return "cos(0.3 + " + " + ".join(f"{float(c[j])!r}*x[{j + 1}]" for j in range(d)) + ")"
    return "exp(-(" + " + ".join(f"{float(c[j]) ** 2!r}*(x[{j + 1}] - {float(w[j])!r})^2" for j in range(d)) + "))"


fams = sys.argv[1].split(",") if len(sys.argv) > 1 else ["expabs"]
ds = [int(v) for v in sys.argv[2].split(",")] if len(sys.argv) > 2 else [16, 24, 32, 48, 64, 96, 128]
ns = [int(v) for v in sys.argv[3].split(",")] if len(sys.argv) > 3 else [2147483647, 16777213, 1000003]
A = {2147483647: 1440510675, 16777213: 1234567, 1000003: 76231}
for n in ns:
    a = A.get(n, 76231)
    for fam in fams:
        for d in ds:
            rng = np.random.default_rng(d)
            f = lq.parse(text_of(fam, d, rng), d)
            rule = lq.korobov_vector(a, n, d)
            pi = engine.plain_integrand(f, d)
            z = rule.z_reduced_array()
            tf, lf, sf = kernel_ms(pi, n, z, "always")
            td, ld, sd = kernel_ms(pi, n, z, "0")
            print(f"{fam:7s} n={n} d={d:4d}  fft(mode {lf}) {tf:8.3f} ms   direct(mode {ld}) {td:8.3f} ms   "
                  f"ratio {td / tf:5.2f}  rel diff {abs(sf - sd) / abs(sd):.1e}", flush=True)
