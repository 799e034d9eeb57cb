"""n = 2^31 Korobov rule with config 5's integrand: 2^k level layout vs the
mirror-paired index kernel (kernel ms summed over all launches = wall-ish)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_08867_b200 as lq
from paper_2404_08867_b200 import _native as N, engine
from paper_2404_08867_b200.configs import make_config
import torch
cfg = make_config(5)
f = lq.parse(cfg.text, cfg.d)
for k in (24, 31):
    n = 1 << k
    rule = lq.korobov_vector((cfg.plain_a | 1) % n, n, cfg.d)
    z = rule.z_reduced_array(); pi = engine.plain_integrand(f, cfg.d)
    for mode in ("1", "0"):
        os.environ["LQ_ORBIT"] = mode
        lay = N.lattice_layout(pi.struct, n, z)
        s = engine.lattice_sum(pi, n, z)
        torch.cuda.synchronize()
        best = 1e30
        for _ in range(3):
            t0 = time.perf_counter(); engine.lattice_sum(pi, n, z); best = min(best, time.perf_counter() - t0)
        print(f"k={k} LQ_ORBIT={mode} mode={lay.mode} tiles/units={lay.n_units}: {best*1e3:.3f} ms wall  "
              f"{n / best:.3e} pts/s  sum {s!r}", flush=True)
