"""End-to-end slr_integrate times of the small BASELINE configs (1-3) and
mdi_lr of configs 1/2/4/5 (best of 20 after a warm-up)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_08867_b200 as lq
from paper_2404_08867_b200.configs import make_config
for cid in (1, 2, 3):
    c = make_config(cid); f = lq.parse(c.text, c.d); r = lq.korobov_vector(c.plain_a, c.plain_n, c.d)
    lq.slr_integrate(f, r); ts = []
    for _ in range(20):
        t0 = time.perf_counter(); lq.slr_integrate(f, r); ts.append(time.perf_counter() - t0)
    print(f"slr cfg{cid}: {min(ts) * 1e3:.4f} ms")
for cid in (1, 2, 4, 5):
    c = make_config(cid); g = lq.parse(c.text, c.d)
    cfg = lq.MdiConfig(direct_cap=10**10) if cid == 1 else None
    lq.mdi_lr(g, c.d, c.mdi_a, c.mdi_n, cfg=cfg); ts = []
    for _ in range(20):
        t0 = time.perf_counter(); lq.mdi_lr(g, c.d, c.mdi_a, c.mdi_n, cfg=cfg); ts.append(time.perf_counter() - t0)
    print(f"mdi cfg{cid}: {min(ts) * 1e3:.4f} ms")
