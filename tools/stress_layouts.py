import sys, math, os, zlib
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import numpy as np
import paper_2404_08867_b200 as lq
from paper_2404_08867_b200 import engine, _native as N
from test_gpu_orbit import _family_text
import sympy
rng = np.random.default_rng(99)
fams = ["exp", "sincos", "expabs", "pow", "gauss", "qtrig"]
bad = 0; modes = {}
for trial in range(240):
    kind = trial % 3
    if kind == 0:
        n = int(sympy.nextprime(int(rng.integers(1 << 16, 1 << 26))))
    elif kind == 1:
        n = 1 << int(rng.integers(12, 26))
    else:
        n = int(rng.integers(1 << 16, 1 << 24)) | 1
    a = int(rng.integers(2, n - 1)) | (1 if kind == 1 else 0)
    d = int(rng.choice([3, 17, 60, 128, 300, 700]))
    fam = fams[trial % 6]
    f = lq.parse(_family_text(fam, d, rng), d)
    rule = lq.korobov_vector(a % n, n, d)
    pi = engine.plain_integrand(f, d)
    z = rule.z_reduced_array()
    os.environ.pop("LQ_ORBIT", None); os.environ.pop("LQ_PAIR", None)
    lay = N.lattice_layout(pi.struct, n, z)
    got = engine.lattice_sum(pi, n, z)
    os.environ["LQ_ORBIT"] = "0"; os.environ["LQ_PAIR"] = "0"
    want = engine.lattice_sum(pi, n, z)
    modes[lay.mode] = modes.get(lay.mode, 0) + 1
    if not math.isclose(got, want, rel_tol=1e-11, abs_tol=1e-9 * n):
        bad += 1
        print("MISMATCH", trial, fam, n, a, d, lay, got, want, flush=True)
print("done", bad, "mismatches; modes", modes)
