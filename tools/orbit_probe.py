"""Orbit vs index kernels on the plain-sum configs: kernel ms (CUDA events in
liblq) and wall ms of engine.lattice_sum.  Not the bench contract."""

import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2404_08867_b200 as lq  # noqa: E402
from paper_2404_08867_b200 import _native as N, engine  # noqa: E402
from paper_2404_08867_b200.configs import make_config  # noqa: E402


def main():
    h = N.lib()
    ctx = N.ctx()
    N.check(h.lq_ctx_enable_timing(ctx, 1))
    cids = [int(c) for c in (sys.argv[1:] or ["1", "2", "3", "5"])]
    for cid in cids:
        cfg = make_config(cid)
        f = lq.parse(cfg.text, cfg.d)
        rule = lq.korobov_vector(cfg.plain_a, cfg.plain_n, cfg.d)
        z = rule.z_reduced_array()
        pi = engine.plain_integrand(f, cfg.d)
        res = {}
        for mode in ("0", "always"):
            os.environ["LQ_ORBIT"] = mode
            lay = N.lattice_layout(pi.struct, rule.n, z)
            engine.lattice_sum(pi, rule.n, z)
            best_k, best_w = 1e30, 1e30
            for _ in range(5 if cid != 5 else 2):
                t0 = time.perf_counter()
                s = engine.lattice_sum(pi, rule.n, z)
                w = time.perf_counter() - t0
                kms, nl = C.c_float(), C.c_int64()
                N.check(h.lq_last_kernel_ms(ctx, C.byref(kms), C.byref(nl)))
                best_k, best_w = min(best_k, kms.value), min(best_w, w * 1e3)
            res[mode] = s
            print(f"cfg{cid} {pi.kind} n={rule.n} d={cfg.d} LQ_ORBIT={mode:6s} mode={lay.mode} units={lay.n_units} "
                  f"kernel {best_k:.4f} ms  wall {best_w:.4f} ms  pts/s {rule.n / (best_k * 1e-3):.3e}  sum {s!r}",
                  flush=True)
        print(f"cfg{cid} rel diff {abs(res['0'] - res['always']) / abs(res['0']):.2e}")


if __name__ == "__main__":
    main()
