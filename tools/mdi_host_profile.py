"""Where MDI-LR time-to-solution goes on the host (cProfile over repeated
mdi_lr calls of configs 1/2/4/5 after warm-up)."""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_08867_b200 as lq  # noqa: E402
from paper_2404_08867_b200.configs import make_config  # noqa: E402

for cid in (1, 2, 4, 5):
    cfg = make_config(cid)
    g = lq.parse(cfg.text, cfg.d)
    mc = lq.MdiConfig(direct_cap=10**10) if cid == 1 else None
    lq.mdi_lr(g, cfg.d, cfg.mdi_a, cfg.mdi_n, cfg=mc)
    ts = []
    for _ in range(50):
        t0 = time.perf_counter()
        lq.mdi_lr(g, cfg.d, cfg.mdi_a, cfg.mdi_n, cfg=mc)
        ts.append(time.perf_counter() - t0)
    print(f"cfg{cid}: best {min(ts) * 1e3:.3f} ms, median {sorted(ts)[25] * 1e3:.3f} ms")
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(200):
        lq.mdi_lr(g, cfg.d, cfg.mdi_a, cfg.mdi_n, cfg=mc)
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(14)
