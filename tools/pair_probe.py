"""Mirror-paired vs plain per-index kernels on non-Korobov rules (kernel ms)."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import paper_2404_08867_b200 as lq
from paper_2404_08867_b200 import _native as N, engine
from test_gpu_orbit import _family_text, _unit_vector
h = N.lib(); ctx = N.ctx(); N.check(h.lq_ctx_enable_timing(ctx, 1))
for fam, n, d in (("expabs", 2**31 - 1, 1000), ("gauss", 2**27, 300), ("sincos", 2**27, 100)):
    rng = np.random.default_rng(5)
    f = lq.parse(_family_text(fam, d, rng), d)
    rule = lq.LatticeRule(n, _unit_vector(n, d, rng))
    pi = engine.plain_integrand(f, d); z = rule.z_reduced_array()
    res = {}
    for mode in ("1", "0"):
        os.environ["LQ_PAIR"] = mode
        engine.lattice_sum(pi, n, z)
        best = 1e30
        for _ in range(3):
            s = engine.lattice_sum(pi, n, z)
            kms, nl = C.c_float(), C.c_int64(); N.check(h.lq_last_kernel_ms(ctx, C.byref(kms), C.byref(nl)))
            best = min(best, kms.value)
        res[mode] = s
        lay = N.lattice_layout(pi.struct, n, z)
        print(f"{fam} n={n} d={d} LQ_PAIR={mode} mode={lay.mode} kernel {best:.3f} ms  {n / (best * 1e-3):.3e} pts/s"
              f"  {n * d / (best * 1e-3):.3e} pd/s", flush=True)
    print(f"  rel diff {abs(res['1'] - res['0']) / abs(res['0']):.2e}")
