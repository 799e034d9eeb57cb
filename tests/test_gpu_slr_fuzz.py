"""GPU: full plain sums of the reference-frozen expression corpus
(tests/golden/slr_fuzz.json, make_golden.py --only slr_fuzz): every accepted
text of the parser corpus plus random members of the closed families, on
Korobov rules over a prime (orbit / FFT-form layouts), over n = 2^12
(lattice-sequence levels) and a composite n, and on a random z -- the whole
front end (parse, family recognition, bytecode or JIT) and the sum kernels
against the reference's slr_integrate (quad.py:96-104).  Tolerance 1e-10
relative to max(|value|, mean |f|)."""

import math

import pytest

from conftest import load_golden, unhex

pytestmark = pytest.mark.gpu

CASES = load_golden("slr_fuzz")


def test_slr_fuzz_matches_reference():
    import paper_2404_08867_b200 as lq
    from paper_2404_08867_b200 import _native as N, engine
    bad, modes = [], set()
    for c in CASES:
        f = lq.parse(c["text"], c["d"])
        rule = lq.LatticeRule(c["n"], tuple(int(v) for v in c["z"]))
        pi = engine.plain_integrand(f, c["d"])
        modes.add(N.lattice_layout(pi.struct, rule.n, rule.z_reduced_array())[3])
        got = lq.slr_integrate(f, rule).value
        want, scale = unhex(c["value"]), unhex(c["scale"])
        if not (got == want or abs(got - want) <= 1e-10 * max(abs(want), scale)):
            bad.append((c["text"][:60], c["d"], c["n"], c["kind"], got, want))
    assert not bad, bad[:10]
    assert len(CASES) > 300
    # every reduction layout met the reference: per-index, mirror pairs,
    # Korobov orbits (direct and FFT form), 2^k lattice-sequence levels
    assert modes >= {N.LAYOUT_INDEX, N.LAYOUT_PAIRED, N.LAYOUT_ORBIT, N.LAYOUT_ORBIT_FFT, N.LAYOUT_ORBIT_POW2}, modes
