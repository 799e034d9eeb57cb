"""Quick GPU probe: FP64 peak, per-config plain-sum kernel throughput, MDI-LR
time-to-solution.  Prints one line per measurement (not the bench contract)."""

import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import paper_2404_08867_b200 as lq  # noqa: E402
from paper_2404_08867_b200 import _native as N, engine  # noqa: E402
from paper_2404_08867_b200.configs import make_config  # noqa: E402

FLOPS_PER_PD = {1: 2, 2: 3, 3: 5, 5: 3}


def main():
    h = N.lib()
    ctx = N.ctx()
    tf = C.c_double()
    ms = C.c_float()
    for it in (2000, 20000):
        N.check(h.lq_fp64_peak(ctx, it, C.byref(tf), C.byref(ms)))
        print(f"fp64_peak iters={it}: {tf.value:.2f} TFLOP/s ({ms.value:.2f} ms)")
    N.check(h.lq_ctx_enable_timing(ctx, 1))
    for cid in (1, 2, 3, 5):
        cfg = make_config(cid)
        f = lq.parse(cfg.text, cfg.d)
        rule = lq.korobov_vector(cfg.plain_a, cfg.plain_n, cfg.d)
        for force in (False, True, "jit"):
            if force and cid == 5:
                continue
            if force == "jit":
                os.environ["LQ_JIT"] = "always"
                engine._plain_cache.clear()
            else:
                os.environ["LQ_JIT"] = "0"
                engine._plain_cache.clear()
            pi = engine.plain_integrand(f, cfg.d, force_program=bool(force))
            z = rule.z_reduced_array()
            n = rule.n
            end = n if cid != 5 else n
            engine.lattice_sum(pi, n, z, 0, end)
            times = []
            for _ in range(3):
                t0 = time.perf_counter()
                s = engine.lattice_sum(pi, n, z, 0, end)
                wall = time.perf_counter() - t0
                kms = C.c_float()
                nl = C.c_int64()
                N.check(h.lq_last_kernel_ms(ctx, C.byref(kms), C.byref(nl)))
                times.append((kms.value, wall))
            kms = min(t[0] for t in times)
            wall = min(t[1] for t in times)
            pts = end
            pd = pts * cfg.d
            fl = (FLOPS_PER_PD[cid] * cfg.d + 2) * pts
            kind = pi.kind + ("+jit" if pi.struct.prog.jit and pi.family is None else "")
            print(f"cfg{cid} {kind:10s} n={n} d={cfg.d}: kernel {kms:.3f} ms wall {wall*1e3:.3f} ms "
                  f"{pts/kms*1e3:.3e} pts/s {pd/kms*1e3:.3e} pd/s {fl/kms*1e-9:.2f} TF-direct-equiv  value={s/n!r}")
    # steady-state rate of the Gaussian family kernel on a large lattice
    cfg = make_config(3)
    f = lq.parse(cfg.text, cfg.d)
    big = lq.korobov_vector(cfg.plain_a, 2**31 - 1, cfg.d)
    pi = engine.plain_integrand(f, cfg.d)
    engine.lattice_sum(pi, big.n, big.z_reduced_array(), 0, 1 << 27)
    engine.lattice_sum(pi, big.n, big.z_reduced_array(), 0, 1 << 27)
    kms = C.c_float(); nl = C.c_int64()
    N.check(h.lq_last_kernel_ms(ctx, C.byref(kms), C.byref(nl)))
    pd = (1 << 27) * cfg.d
    print(f"quad_exp big-n d=300 2^27 pts: kernel {kms.value:.3f} ms {pd/kms.value*1e3:.3e} pd/s "
          f"{(5*cfg.d+2)*(1<<27)/kms.value*1e-9:.2f} TF")
    for cid, cap in ((2, None), (4, None), (1, 10**10), (5, None)):
        cfg = make_config(cid)
        f = lq.parse(cfg.text, cfg.d)
        mc = lq.MdiConfig(direct_cap=cap) if cap else None
        lq.mdi_lr(f, cfg.d, cfg.mdi_a, cfg.mdi_n, cfg=mc)
        ts = []
        for _ in range(5):
            t0 = time.perf_counter()
            v, rep = lq.mdi_lr(f, cfg.d, cfg.mdi_a, cfg.mdi_n, cfg=mc, with_report=True)
            ts.append(time.perf_counter() - t0)
        print(f"mdi cfg{cid}: {min(ts)*1e3:.3f} ms value={v!r} raw={rep.value!r} log_raw={rep.log_raw!r}")


if __name__ == "__main__":
    main()
