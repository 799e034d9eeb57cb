"""cProfile of repeated mdi_lr calls (host-side time-to-solution breakdown)."""
import cProfile, os, pstats, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_08867_b200 as lq
from paper_2404_08867_b200.configs import make_config
for cid in (int(x) for x in (sys.argv[1:] or ["4", "5"])):
    mc = make_config(cid)
    g = lq.parse(mc.text, mc.d)
    mcfg = lq.MdiConfig(direct_cap=10**10) if cid == 1 else None
    lq.mdi_lr(g, mc.d, mc.mdi_a, mc.mdi_n, cfg=mcfg)
    t0 = time.perf_counter()
    for _ in range(50):
        lq.mdi_lr(g, mc.d, mc.mdi_a, mc.mdi_n, cfg=mcfg, with_report=True)
    print(f"cfg{cid}: {(time.perf_counter() - t0) / 50 * 1e3:.3f} ms per call")
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(50):
        lq.mdi_lr(g, mc.d, mc.mdi_a, mc.mdi_n, cfg=mcfg, with_report=True)
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(14)
