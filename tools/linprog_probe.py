"""Kernel time of a function of one linear form outside the closed families
(1/(1 + (2L - 0.8)^2), d = 1000, config 5's lattice): FFT-form chains with the
bytecode outer vs the per-index bytecode kernel (on a 2^24-point sub-range,
scaled)."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2404_08867_b200 as lq
from paper_2404_08867_b200 import _native as N, engine
from paper_2404_08867_b200.configs import make_config
cfg = make_config(5)
d = cfg.d
c = np.asarray(cfg.c) / 10.0
L = " + ".join(f"{float(v)!r}*x[{j + 1}]" for j, v in enumerate(c))
f = lq.parse(f"1/(1 + (2*({L}) - 0.8)^2)", d)
rule = lq.korobov_vector(cfg.plain_a, cfg.plain_n, d)
z = rule.z_reduced_array()
pi = engine.plain_integrand(f, d)
h, ctx = N.lib(), N.ctx()
N.check(h.lq_ctx_enable_timing(ctx, 1))
def kernel_ms(lo, hi):
    best = 1e30
    for _ in range(3):
        s = engine.lattice_sum(pi, rule.n, z, lo, hi)
        kms, nl = C.c_float(), C.c_int64()
        N.check(h.lq_last_kernel_ms(ctx, C.byref(kms), C.byref(nl)))
        best = min(best, kms.value)
    return best, s
print(pi.kind, N.lattice_layout(pi.struct, rule.n, z).mode)
full, s_full = kernel_ms(0, rule.n)
sub, _ = kernel_ms(0, 1 << 24)
print(f"FFT form (program outer): {full:.2f} ms for n = 2^31 - 1 ({rule.n / full / 1e-3:.3e} pts/s); "
      f"per-index bytecode: {sub:.2f} ms per 2^24 points -> {sub * rule.n / (1 << 24):.0f} ms extrapolated; "
      f"estimate {s_full / rule.n!r}")
