"""GPU: concurrent callers.  include/lq.h's contract is one context per device
per thread (_native.ctx keys contexts by thread), thread-local errors, and
process-wide plan caches behind mutexes.  Four threads run the same mix of
plain sums (family, orbit, FFT-form and composite-n layouts), points blocks
and MDI-LR at once -- ctypes drops the GIL inside every liblq call, so the C
side really runs in parallel -- and every result must equal the serial one bit
for bit (the sums are order-fixed, so a race shows up as a different value)."""

import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _jobs():
    import paper_2404_08867_b200 as lq
    from paper_2404_08867_b200.configs import make_config

    jobs = []
    for k in (1, 2, 3):
        cfg = make_config(k)
        f = lq.parse(cfg.text, cfg.d)
        rule = lq.korobov_vector(cfg.plain_a, cfg.plain_n, cfg.d)
        jobs.append((f"slr cfg{k}", lambda f=f, rule=rule: lq.slr_integrate(f, rule).value))
    rng = np.random.default_rng(7)
    d = 64
    c = rng.uniform(0.0, 1.0, d)
    c *= 10.0 / c.sum()
    text = "exp(-abs(" + " + ".join(f"{float(v)!r}*(x[{j + 1}] - 0.5)" for j, v in enumerate(c)) + "))"
    f64 = lq.parse(text, d)
    for n, a in ((4194319, 1234567), (4194304 * 3 + 10, 1000003)):   # prime (FFT form), composite
        rule = lq.korobov_vector(a, n, d)
        jobs.append((f"slr d=64 n={n}", lambda f=f64, rule=rule: lq.slr_integrate(f, rule).value))
    rule5 = lq.korobov_vector(17, 100003, 5)
    jobs.append(("points", lambda: lq.points_block(rule5, 1000, 3000).tobytes()))
    g = lq.parse("exp(-sum(i=1..d, x[i]^2)/2)", 8)
    jobs.append(("mdi", lambda: lq.mdi_lr(g, 8, 5, 5**8)))
    inv = lq.parse("(1 + sum(i=1..d, x[i]))^(-(d+1))", 6)
    jobs.append(("mdi linform", lambda: lq.mdi_lr(inv, 6, 4, 4**6 + 1)))
    return jobs


def test_threads_match_serial():
    jobs = _jobs()
    serial = {name: fn() for name, fn in jobs}
    results, errors = [], []

    def worker(seed):
        order = list(range(len(jobs)))
        np.random.default_rng(seed).shuffle(order)
        try:
            for _ in range(3):
                for i in order:
                    name, fn = jobs[i]
                    results.append((name, fn()))
        except Exception as e:   # surfaced below with the thread's traceback text
            errors.append(repr(e))

    threads = [threading.Thread(target=worker, args=(s,)) for s in range(4)]
    for t in threads:
        t.start()
    for t in threads:
        t.join(timeout=600)
    assert not any(t.is_alive() for t in threads), "a worker hung"
    assert not errors, errors
    assert len(results) == 4 * 3 * len(jobs)
    for name, got in results:
        assert got == serial[name], (name, got, serial[name])


def test_cold_plans_built_concurrently():
    # four threads plan the same fresh lattices at the same time (orbit plans
    # for prime n, divisor-class plans for composite n are built under the
    # planners' mutexes); the cached plans must still cover every index once
    # and every thread must get the oracle's sum
    import ctypes as C

    import paper_2404_08867_b200 as lq
    from oracle import np_oracle as orc
    from paper_2404_08867_b200 import _native as N, engine

    d = 128   # the FFT form from d = 112 at these n (fft_min_d), so FFT plans too
    rng = np.random.default_rng(11)
    c = rng.uniform(0.0, 1.0, d)
    c *= 8.0 / c.sum()
    text = "exp(-abs(" + " + ".join(f"{float(v)!r}*(x[{j + 1}] - 0.25)" for j, v in enumerate(c)) + "))"
    f = lq.parse(text, d)
    cases = [(1000231, 7919), (999999, 1013), (1 << 20, 12345), (1048583, 99991)]   # prime, composite, 2^k, prime
    rules = [lq.korobov_vector(a, n, d) for n, a in cases]
    barrier = threading.Barrier(4)
    results, errors = {}, []

    def worker(t):
        try:
            barrier.wait()
            for i in range(len(rules)):
                rule = rules[(i + t) % len(rules)] if t % 2 else rules[i]
                results[(t, rule.n)] = lq.slr_integrate(f, rule).value
        except Exception as e:
            errors.append(repr(e))

    threads = [threading.Thread(target=worker, args=(t,)) for t in range(4)]
    for t in threads:
        t.start()
    for t in threads:
        t.join(timeout=600)
    assert not errors, errors
    pi = engine.plain_integrand(f, d)
    h = N.lib()
    for rule in rules:
        vals = {results[(t, rule.n)] for t in range(4)}
        assert len(vals) == 1, (rule.n, vals)
        z = rule.z_reduced_array()
        miss, rep = C.c_int64(), C.c_int64()
        N.check(h.lq_layout_cover(C.byref(pi.struct), rule.n, N.as_ptr(z), C.byref(miss), C.byref(rep)))
        assert (miss.value, rep.value) == (0, 0), rule.n
        want = orc.slr_value(text, rule.n, rule.z)
        got = vals.pop()
        assert abs(got - want) <= 1e-10 * abs(want), (rule.n, got, want)
