"""Latency of the public API vs the bare C call for the small configs."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_08867_b200 as lq  # noqa: E402
from paper_2404_08867_b200 import _native as N, engine  # noqa: E402
from paper_2404_08867_b200.configs import make_config  # noqa: E402


def best(fn, k=200):
    fn()
    ts = []
    for _ in range(k):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return min(ts) * 1e6, sorted(ts)[k // 2] * 1e6


for cid in (1, 2, 3):
    cfg = make_config(cid)
    f = lq.parse(cfg.text, cfg.d)
    rule = lq.korobov_vector(cfg.plain_a, cfg.plain_n, cfg.d)
    pi = engine.plain_integrand(f, cfg.d)
    z = rule.z_reduced_array()
    h, ctx, out = N.lib(), N.ctx(), C.c_double()
    api = best(lambda: lq.slr_integrate(f, rule))
    bare = best(lambda: h.lq_lattice_sum(ctx, C.byref(pi.struct), rule.n, N.as_ptr(z), 0, rule.n, C.byref(out)))
    h.lq_ctx_enable_timing(ctx, 1)
    h.lq_lattice_sum(ctx, C.byref(pi.struct), rule.n, N.as_ptr(z), 0, rule.n, C.byref(out))
    kms, nl = C.c_float(), C.c_int64()
    h.lq_last_kernel_ms(ctx, C.byref(kms), C.byref(nl))
    h.lq_ctx_enable_timing(ctx, 0)
    print(f"cfg{cid}: api best/median {api[0]:.1f}/{api[1]:.1f} us, bare C call {bare[0]:.1f}/{bare[1]:.1f} us, "
          f"kernel {kms.value * 1e3:.1f} us ({nl.value} launches)")
