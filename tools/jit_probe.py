import os, sys, time
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
os.environ["LQ_FFT"] = "0"
import fft_cases
import paper_2404_08867_b200 as lq
from paper_2404_08867_b200 import engine
key, text, _, n, a = fft_cases.linprog_case("recip_sq", 1000003, 1000)
d = 1000
f = lq.parse(text, d)
rule = lq.korobov_vector(a, n, d)
pi = engine.plain_integrand(f, d)
t = time.time(); s = engine.lattice_sum(pi, n, rule.z_reduced_array()); print("first", time.time() - t, s)
t = time.time(); s = engine.lattice_sum(pi, n, rule.z_reduced_array()); print("second", time.time() - t, s)
os.environ["LQ_JIT"] = "0"
pi2 = engine.plain_integrand(f, d, force_program=True)
t = time.time(); s = engine.lattice_sum(pi2, n, rule.z_reduced_array()); print("interp", time.time() - t, s)
