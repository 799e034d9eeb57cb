import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_08867_b200 as lq
from paper_2404_08867_b200 import _native as N, engine
from paper_2404_08867_b200.configs import make_config
h = N.lib(); ctx = N.ctx()
N.check(h.lq_ctx_enable_timing(ctx, 1))
cfg = make_config(3)
f = lq.parse(cfg.text, cfg.d)
for n, npts in ((2**31 - 1, 1 << 27), (cfg.plain_n, cfg.plain_n)):
    rule = lq.korobov_vector(cfg.plain_a, n, cfg.d)
    pi = engine.plain_integrand(f, cfg.d)
    best = 1e9
    for _ in range(4):
        s = engine.lattice_sum(pi, n, rule.z_reduced_array(), 0, npts)
        kms = C.c_float(); nl = C.c_int64()
        N.check(h.lq_last_kernel_ms(ctx, C.byref(kms), C.byref(nl)))
        best = min(best, kms.value)
    print(os.environ.get("LQ_LIB_PATH", "default"), n, f"{best:.3f} ms {npts*cfg.d/best*1e3:.3e} pd/s value={s/npts!r}")
