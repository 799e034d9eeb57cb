"""Host overhead of one slr_integrate call on cfg5 (wall time per call and a cProfile of 10 calls)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import time, cProfile, pstats, torch
import paper_2404_08867_b200 as lq
from paper_2404_08867_b200.configs import make_config
cfg = make_config(5)
f = lq.parse(cfg.text, cfg.d)
rule = lq.korobov_vector(cfg.plain_a, cfg.plain_n, cfg.d)
lq.slr_integrate(f, rule); torch.cuda.synchronize()
ts=[]
for _ in range(10):
    t0=time.perf_counter(); lq.slr_integrate(f, rule); ts.append(time.perf_counter()-t0)
print("e2e ms", [round(t*1e3,3) for t in ts])
pr=cProfile.Profile(); pr.enable()
for _ in range(10): lq.slr_integrate(f, rule)
pr.disable()
pstats.Stats(pr).sort_stats('tottime').print_stats(12)
