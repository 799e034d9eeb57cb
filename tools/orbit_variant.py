"""Time the cfg5 orbit kernel of the liblq variant named by LQ_LIB_PATH."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_08867_b200 as lq
from paper_2404_08867_b200 import _native as N, engine
from paper_2404_08867_b200.configs import make_config
h = N.lib(); ctx = N.ctx(); N.check(h.lq_ctx_enable_timing(ctx, 1))
cfg = make_config(int(sys.argv[1]) if len(sys.argv) > 1 else 5)
f = lq.parse(cfg.text, cfg.d); rule = lq.korobov_vector(cfg.plain_a, cfg.plain_n, cfg.d)
z = rule.z_reduced_array(); pi = engine.plain_integrand(f, cfg.d)
os.environ["LQ_ORBIT"] = "always"
engine.lattice_sum(pi, rule.n, z)
best = 1e30
for _ in range(4):
    s = engine.lattice_sum(pi, rule.n, z)
    kms, nl = C.c_float(), C.c_int64(); N.check(h.lq_last_kernel_ms(ctx, C.byref(kms), C.byref(nl)))
    best = min(best, kms.value)
print(f"{os.path.basename(N.LIB_PATH)} cfg{cfg.cid if hasattr(cfg,'cid') else ''} kernel {best:.3f} ms  {rule.n / (best * 1e-3):.4e} pts/s  sum {s!r}", flush=True)
