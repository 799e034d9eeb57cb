import ctypes as C, sys, os, time
sys.path.insert(0, os.getcwd())
import paper_2404_08867_b200 as lq
from paper_2404_08867_b200 import _native as N, engine
from paper_2404_08867_b200.configs import make_config
h = N.lib(); ctx = N.ctx(); N.check(h.lq_ctx_enable_timing(ctx, 1))
mc = make_config(5); g = lq.parse(mc.text, mc.d)
for _ in range(3): lq.mdi_lr(g, mc.d, mc.mdi_a, mc.mdi_n)
kms, nl = C.c_float(), C.c_int64(); N.check(h.lq_last_kernel_ms(ctx, C.byref(kms), C.byref(nl)))
fam = engine.plain_family(g, mc.d)
_, _, wn, ww, nn = engine._cf_inputs(fam.beta, (mc.mdi_a,)*mc.d, fam.alpha, fam.kappa)
print("cfg5 mdi kernel ms", kms.value, "launches", nl.value, "nodes", nn, "n_w", len(wn))
