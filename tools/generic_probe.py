"""Throughput of the generic (bytecode / NVRTC JIT) plain-sum kernels on
corpus-style integrands outside the closed families."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_08867_b200 as lq
from paper_2404_08867_b200 import _native as N, engine, corpus
from paper_2404_08867_b200.configs import make_config
h = N.lib(); ctx = N.ctx(); N.check(h.lq_ctx_enable_timing(ctx, 1))
cases = [("ratprod d=100", corpus.corpus_expr("ratprod", 100), 100, 1 << 22),
         ("expxy d=2", corpus.corpus_expr("expxy", 2), 2, 1 << 26)]
cfg4 = make_config(4)
cases.append(("cfg4 product peak d=500", lq.parse(cfg4.text, cfg4.d), cfg4.d, 1 << 20))
for name, f, d, n in cases:
    rule = lq.korobov_vector(3, n + 1 if n % 2 == 0 else n, d)
    z = rule.z_reduced_array()
    for mode in ("0", "always"):
        os.environ["LQ_JIT"] = mode
        engine._plain_cache.clear()
        pi = engine.plain_integrand(f, d)
        engine.lattice_sum(pi, rule.n, z)
        best = 1e30
        for _ in range(3):
            engine.lattice_sum(pi, rule.n, z)
            kms, nl = C.c_float(), C.c_int64(); N.check(h.lq_last_kernel_ms(ctx, C.byref(kms), C.byref(nl)))
            best = min(best, kms.value)
        print(f"{name} n={rule.n} LQ_JIT={mode}: {best:.3f} ms  {rule.n / best * 1e3:.3e} pts/s  "
              f"{rule.n * d / best * 1e3:.3e} pd/s", flush=True)
