import os, sys
sys.path.insert(0, "/root/repo")
import paper_2404_08867_b200 as lq
from paper_2404_08867_b200.configs import make_config
for cid in (1, 2):
    cfg = make_config(cid)
    f = lq.parse(cfg.text, cfg.d)
    rule = lq.korobov_vector(cfg.plain_a, cfg.plain_n, cfg.d)
    for _ in range(3):
        lq.slr_integrate(f, rule)
