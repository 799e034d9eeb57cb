import ctypes as C, os, sys
sys.path.insert(0, '/root/repo')
import paper_2404_08867_b200 as lq
from paper_2404_08867_b200 import _native as N, engine, corpus
from paper_2404_08867_b200.configs import make_config
h = N.lib(); ctx = N.ctx(); N.check(h.lq_ctx_enable_timing(ctx, 1))
cfg4 = make_config(4)
for name, f, d, n in (("ratprod", corpus.corpus_expr("ratprod", 100), 100, 2**27 - 39), ("cfg4", lq.parse(cfg4.text, cfg4.d), 500, 2**25 - 39)):
    for mode in ("0", "1"):
        os.environ["LQ_ORBIT"] = mode
        rule = lq.korobov_vector(3, n, d); z = rule.z_reduced_array(); pi = engine.plain_integrand(f, d)
        lay = N.lattice_layout(pi.struct, n, z)
        s = engine.lattice_sum(pi, n, z); best = 1e30
        for _ in range(3):
            engine.lattice_sum(pi, n, z); kms, nl = C.c_float(), C.c_int64(); N.check(h.lq_last_kernel_ms(ctx, C.byref(kms), C.byref(nl))); best = min(best, kms.value)
        print(name, pi.kind, n, d, f"LQ_ORBIT={mode} mode={lay.mode}", f"{best:.3f} ms {n*d/best*1e3:.3e} pd/s sum {s!r}")
