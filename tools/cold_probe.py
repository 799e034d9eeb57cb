"""Break down the cold first call of slr_integrate(config 5) in a fresh process."""
import os
import sys
import time

t00 = time.perf_counter()
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_08867_b200 as lq  # noqa: E402
from paper_2404_08867_b200 import _native as N, engine  # noqa: E402
from paper_2404_08867_b200.configs import make_config  # noqa: E402

t0 = time.perf_counter()
N.ctx()
t1 = time.perf_counter()
cfg = make_config(5)
f = lq.parse(cfg.text, cfg.d)
t2 = time.perf_counter()
rule = lq.korobov_vector(cfg.plain_a, cfg.plain_n, cfg.d)
pi = engine.plain_integrand(f, cfg.d)
t3 = time.perf_counter()
lay = N.lattice_layout(pi.struct, rule.n, rule.z_reduced_array())
t4 = time.perf_counter()
v = lq.slr_integrate(f, rule).value
t5 = time.perf_counter()
v2 = lq.slr_integrate(f, rule).value
t6 = time.perf_counter()
print(f"imports {t0 - t00:.3f}s ctx {1e3 * (t1 - t0):.1f} ms parse {1e3 * (t2 - t1):.1f} ms "
      f"lower {1e3 * (t3 - t2):.1f} ms layout(plan) {1e3 * (t4 - t3):.1f} ms first call {1e3 * (t5 - t4):.1f} ms "
      f"second call {1e3 * (t6 - t5):.1f} ms")
