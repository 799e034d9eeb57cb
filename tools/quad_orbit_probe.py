"""Gaussian family (config 3's integrand, d = 300) on a full Korobov lattice of
~2^27 points: orbit vs mirror-paired vs plain index kernels (kernel ms)."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_08867_b200 as lq
from paper_2404_08867_b200 import _native as N, engine
from paper_2404_08867_b200.configs import make_config
h = N.lib(); ctx = N.ctx(); N.check(h.lq_ctx_enable_timing(ctx, 1))
cfg = make_config(3)
f = lq.parse(cfg.text, cfg.d)
n = 134217689                      # prime just below 2^27
rule = lq.korobov_vector(cfg.plain_a % n, n, cfg.d)
z = rule.z_reduced_array()
pi = engine.plain_integrand(f, cfg.d)
for orb, pair in (("1", "1"), ("0", "1"), ("0", "0")):
    os.environ["LQ_ORBIT"], os.environ["LQ_PAIR"] = orb, pair
    lay = N.lattice_layout(pi.struct, n, z)
    s = engine.lattice_sum(pi, n, z)
    best = 1e30
    for _ in range(3):
        engine.lattice_sum(pi, n, z)
        kms, nl = C.c_float(), C.c_int64(); N.check(h.lq_last_kernel_ms(ctx, C.byref(kms), C.byref(nl)))
        best = min(best, kms.value)
    print(f"quad d={cfg.d} n={n} mode={lay.mode}: {best:.3f} ms  {n * cfg.d / best * 1e3:.3e} pd/s  sum {s!r}", flush=True)
