"""Kernel time of every rank's shard of the cfg5 plain sum (P = 1, 2, 4, 8),
run as sequential launches on one GPU: the max over ranks is what a P-GPU
run's kernel phase would take (the tail/balance of the per-rank grids)."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2404_08867_b200 as lq
from paper_2404_08867_b200 import _native as N, engine
from paper_2404_08867_b200.distributed import shard_range
from paper_2404_08867_b200.configs import make_config
h = N.lib(); ctx = N.ctx(); N.check(h.lq_ctx_enable_timing(ctx, 1))
cfg = make_config(int(sys.argv[1]) if len(sys.argv) > 1 else 5)
f = lq.parse(cfg.text, cfg.d); rule = lq.korobov_vector(cfg.plain_a, cfg.plain_n, cfg.d)
z = rule.z_reduced_array(); pi = engine.plain_integrand(f, cfg.d)
S = N.lattice_layout(pi.struct, rule.n, z).n_supers
parts = torch.zeros(S, dtype=torch.float64, device="cuda")
for P in (1, 2, 4, 8):
    worst = 0.0
    for r in range(P):
        lo, hi = shard_range(S, r, P)
        best = 1e30
        for _ in range(3):
            N.check(h.lq_lattice_partials(ctx, C.byref(pi.struct), rule.n, N.as_ptr(z), lo, hi,
                                          C.c_void_p(parts.data_ptr() + 8 * lo)))
            kms, nl = C.c_float(), C.c_int64(); N.check(h.lq_last_kernel_ms(ctx, C.byref(kms), C.byref(nl)))
            best = min(best, kms.value)
        worst = max(worst, best)
    print(f"P={P} max-over-ranks kernel {worst:.3f} ms  (x{P} = {worst * P:.3f} ms; "
          f"strong-scaling kernel efficiency vs P=1 needs the P=1 line)", flush=True)
