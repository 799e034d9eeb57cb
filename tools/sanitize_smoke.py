"""Small invocations of every liblq kernel, for compute-sanitizer memcheck."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2404_08867_b200 as lq  # noqa: E402
from paper_2404_08867_b200 import engine  # noqa: E402
from paper_2404_08867_b200.configs import make_config  # noqa: E402

r = lq.korobov_vector(7, 1009, 5)
lq.points_block(r, 3, 300)
lq.points_block(lq.LatticeRule(2**40 + 15, (1, 3, 5)), 2**35, 2**35 + 100)
for cid in (1, 2, 3):
    cfg = make_config(cid)
    f = lq.parse(cfg.text, cfg.d)
    rule = lq.korobov_vector(cfg.plain_a, cfg.plain_n, cfg.d)
    lq.slr_integrate(f, rule)
    engine.lattice_sum(engine.plain_integrand(f, cfg.d, force_program=True), rule.n, rule.z_reduced_array(), 0, 5000)
cfg = make_config(5)
f = lq.parse(cfg.text, cfg.d)
rule = lq.korobov_vector(cfg.plain_a, cfg.plain_n, cfg.d)
engine.lattice_sum(engine.plain_integrand(f, cfg.d), rule.n, rule.z_reduced_array(), 0, 1 << 16)
lq.slr_integrate(lq.parse("x[2]*exp(x[1]*x[2])", 2), lq.korobov_vector(10, 2**31 + 11, 2))
lq.implr_integrate(lq.parse("(1 + x[1] + x[2] + x[3])^(-4)", 3), 3, 5, 125)
lq.mdi_lr(lq.parse(make_config(2).text, 100), 100, 64, 64**100)
lq.mdi_lr(lq.parse("exp(-abs(" + " + ".join(f"{0.1 + (k * 0.6180339887) % 1.0!r}*x[{k + 1}]" for k in range(40)) + " - 10.0))", 40),
          40, 8, 8**40)
# round 2: level collapse (shared-memory and global levels), cores, sub-grids
inv = lq.parse("(1 + sum(i=1..d, x[i]))^(-(d+1))", 10)
lq.mdi_lr(inv, 10, 8, 8**10 + 1)
os.environ["LQ_LINFORM_SMEM"] = "0"
lq.mdi_lr(inv, 10, 8, 8**10 + 1)
del os.environ["LQ_LINFORM_SMEM"]
lq.mdi_lr(lq.parse("exp(x[1]*x[2])*prod(i=3..d, 1/(1 + x[i]^2))", 8), 8, 6, 6**8)
lq.mdi_lr(lq.parse("exp(x[1]*x[2]*x[3]*x[4])", 8), 8, 4, 4**8)
lq.p_alpha(lq.korobov_vector(76, 1009, 6), 4)
lq.shift_avg_wce_sq(lq.korobov_vector(76, 1009, 6))
lq.cbc_construct(101, 4)
lq.korobov_search(101, 4)
# session 2: eval_array, weighted level collapse, term sums, exact quality sums
f3 = lq.parse("exp(x[1]) * cos(x[2] + 2*x[3])", 3)
lq.eval_array(f3, {1: np.linspace(0, 1, 1000), 2: 0.25, 3: np.linspace(1, 0, 1000)})
w = lq.parse("exp(-sum(i=1..d, x[i]^2))*(1 + sum(i=1..d, x[i]))^(-2)", 8)
lq.mdi_lr(w, 8, 8, 8**8 + 1)
os.environ["LQ_LINFORM_SMEM"] = "0"
lq.mdi_lr(w, 8, 8, 8**8 + 1)
del os.environ["LQ_LINFORM_SMEM"]
lq.mdi_lr(lq.parse("(1 + sum(i=1..d, x[i]))^(-2) + exp(-sum(i=1..d, x[i]^2))", 6), 6, 6, 6**6 + 1)
lq.p_alpha(lq.LatticeRule(1009, (1, 400)), 2)
lq.mdi_lr(lq.parse("(1 + sum(i=1..d, x[i]))^(-2)*(2 + sum(i=1..d, (-1)^i*x[i]))^(-1)", 6), 6, 6, 6**6 + 1)
cfg = make_config(5)
lq.slr_integrate(lq.parse(cfg.text, cfg.d), lq.korobov_vector(12345679, 10**8, cfg.d))
print("sanitize smoke ok")
