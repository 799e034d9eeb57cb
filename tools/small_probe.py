"""Launch-latency probe for the small plain-sum configs (index kernels)."""
import ctypes as C, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_08867_b200 as lq
from paper_2404_08867_b200 import _native as N, engine
from paper_2404_08867_b200.configs import make_config
h = N.lib(); ctx = N.ctx(); N.check(h.lq_ctx_enable_timing(ctx, 1))
for cid in (1, 2):
    cfg = make_config(cid)
    f = lq.parse(cfg.text, cfg.d); rule = lq.korobov_vector(cfg.plain_a, cfg.plain_n, cfg.d)
    z = rule.z_reduced_array(); pi = engine.plain_integrand(f, cfg.d)
    engine.lattice_sum(pi, rule.n, z)
    bk, bw = 1e30, 1e30
    for _ in range(20):
        t0 = time.perf_counter(); engine.lattice_sum(pi, rule.n, z); w = time.perf_counter() - t0
        kms, nl = C.c_float(), C.c_int64(); N.check(h.lq_last_kernel_ms(ctx, C.byref(kms), C.byref(nl)))
        bk, bw = min(bk, kms.value), min(bw, w)
    print(f"{os.path.basename(N.LIB_PATH)} cfg{cid} kernel {bk*1e3:.1f} us wall {bw*1e6:.1f} us", flush=True)
