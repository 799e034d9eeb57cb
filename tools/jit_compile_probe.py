"""NVRTC compile time of jit.compile_expr against expression size."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2404_08867_b200 as lq
from paper_2404_08867_b200 import jit, lower
rng = np.random.default_rng(0)
for d in (8, 32, 64, 128, 256):
    c = rng.uniform(0, 1, d)
    text = "1/(1 + (" + " + ".join(f"{float(c[j]) / d!r}*x[{j + 1}]" for j in range(d)) + ")^2)"
    f = lq.parse(text, d)
    n_insn = len(lower.compile_program(f))
    t = time.time()
    h = jit.compile_expr(f)
    print(f"d={d} insn={n_insn} compile {time.time() - t:.2f} s ok={bool(h)}", flush=True)
