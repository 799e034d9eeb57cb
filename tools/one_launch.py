"""One cfg5 plain-sum launch over a 2^28-point range (for ncu captures)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_08867_b200 as lq
from paper_2404_08867_b200 import engine
from paper_2404_08867_b200.configs import make_config
cid = int(sys.argv[1]) if len(sys.argv) > 1 else 5
npts = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 28
cfg = make_config(cid)
f = lq.parse(cfg.text, cfg.d)
rule = lq.korobov_vector(cfg.plain_a, cfg.plain_n, cfg.d)
pi = engine.plain_integrand(f, cfg.d)
for _ in range(2):
    s = engine.lattice_sum(pi, rule.n, rule.z_reduced_array(), 0, min(npts, rule.n))
print(pi.kind, s)
