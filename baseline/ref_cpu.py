"""The reference arm: latquad itself (installed into baseline/_ref by
``pip install --no-index --no-build-isolation --no-deps --target baseline/_ref``
from a copy of /root/reference/pkg), timed on the host cores of whatever box
runs bench.py.  Nothing here touches the GPU package's kernels; the synthetic
configs come from paper_2404_08867_b200.configs (seeded numpy arrays only).

* ``cfg5_range_sum`` -- config 5's plain sum over an index range: the
  reference's own lattice.points_block (lattice.py:96-105) + its integrand in
  numpy, exp(-|x c - c.w|) (the reference grammar has no |.|,
  exprcore.py:638), in contiguous chunks over worker processes.
* ``suite`` -- the reference's public API as is, one core: slr_integrate on
  configs 1-3 (quad.py:96-104) and mdi_lr on configs 2 and 1 (mdi.py:215-234;
  config 1 with direct_cap = 1e10, which its base sweep needs).
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF = os.path.join(HERE, "_ref")
REPO = os.path.dirname(HERE)


def available():
    return os.path.isdir(os.path.join(REF, "latquad"))


def _import():
    if not available():
        raise ImportError(f"{REF} not installed (see baseline/ref_cpu.py)")
    if REF not in sys.path:
        sys.path.insert(0, REF)
    if REPO not in sys.path:
        sys.path.insert(0, REPO)
    import latquad
    return latquad


def _chunk(args):
    from threadpoolctl import threadpool_limits
    lo, hi = args
    _import()
    from latquad.lattice import LatticeRule, points_block
    from paper_2404_08867_b200.configs import make_config
    cfg = make_config(5)
    rule = LatticeRule(cfg.plain_n, cfg.plain_z())
    c = np.asarray(cfg.c)
    cw = float(np.dot(c, np.asarray(cfg.w)))
    acc = 0.0
    with threadpool_limits(1):
        for start in range(lo, hi, 1 << 12):
            pts = points_block(rule, start, min(start + (1 << 12), hi))
            acc += float(np.sum(np.exp(-np.abs(pts @ c - cw))))
    return acc


def cfg5_range_sum(lo, hi, workers=1):
    """sum over i in [lo, hi) of config 5's integrand at the reference's points."""
    if workers <= 1:
        return _chunk((lo, hi))
    import multiprocessing as mp
    bounds = np.linspace(lo, hi, workers + 1).astype(np.int64)
    with mp.get_context("fork").Pool(workers) as pool:
        return float(sum(pool.map(_chunk, [(int(bounds[k]), int(bounds[k + 1])) for k in range(workers)])))


def suite(mdi_cfg1=True):
    """Seconds of the reference's own API on configs 1-3 (plain) and 2, 1 (MDI-LR), one core."""
    from threadpoolctl import threadpool_limits
    _import()
    from latquad import exprcore
    from latquad.lattice import LatticeRule
    from latquad.mdi import MdiConfig, mdi_lr
    from latquad.quad import slr_integrate
    from paper_2404_08867_b200.configs import make_config
    out = {}
    with threadpool_limits(1):
        for cid in (1, 2, 3):
            cfg = make_config(cid)
            f = exprcore.parse(cfg.text, cfg.d)
            rule = LatticeRule(cfg.plain_n, cfg.plain_z())
            t0 = time.perf_counter()
            r = slr_integrate(f, rule)
            out[f"slr_cfg{cid}_s"] = time.perf_counter() - t0
            out[f"slr_cfg{cid}_value"] = r.value
        for cid in ((2, 1) if mdi_cfg1 else (2,)):
            cfg = make_config(cid)
            f = exprcore.parse(cfg.text, cfg.d)
            mc = MdiConfig(direct_cap=10**10) if cid == 1 else None
            t0 = time.perf_counter()
            v = mdi_lr(f, cfg.d, cfg.mdi_a, cfg.mdi_n, cfg=mc)
            out[f"mdi_cfg{cid}_s"] = time.perf_counter() - t0
            out[f"mdi_cfg{cid}_value"] = v
    return out


if __name__ == "__main__":
    import json
    print(json.dumps(suite("--no-mdi-cfg1" not in sys.argv)))


def suite_one(which):
    """One entry of ``suite`` ('slr1'..'slr3', 'mdi1', 'mdi2'), for a process pool."""
    from threadpoolctl import threadpool_limits
    _import()
    from latquad import exprcore
    from latquad.lattice import LatticeRule
    from latquad.mdi import MdiConfig, mdi_lr
    from latquad.quad import slr_integrate
    from paper_2404_08867_b200.configs import make_config
    cid = int(which[-1])
    cfg = make_config(cid)
    f = exprcore.parse(cfg.text, cfg.d)
    with threadpool_limits(1):
        t0 = time.perf_counter()
        if which.startswith("slr"):
            v = slr_integrate(f, LatticeRule(cfg.plain_n, cfg.plain_z())).value
        else:
            v = mdi_lr(f, cfg.d, cfg.mdi_a, cfg.mdi_n, cfg=MdiConfig(direct_cap=10**10) if cid == 1 else None)
        dt = time.perf_counter() - t0
    return {f"{which[:3]}_cfg{cid}_s": dt, f"{which[:3]}_cfg{cid}_value": v}
