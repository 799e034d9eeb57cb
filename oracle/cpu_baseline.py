"""CPU baseline legs of bench.py (test infrastructure, never the product path).

The reference path for config 5 is lattice.points_block followed by the
integrand (/root/reference/pkg/src/latquad/lattice.py:96-105,
quad.py:96-104); its exp(-|.|) integrand is outside the reference grammar,
so the numpy restatement used for the golden vectors
(tests/golden/make_golden.py, kind "ref_points+numpy") is timed here.
Multi-core runs split the index range into contiguous chunks across
processes, the way SURVEY.md §8(d) item 3 describes.
"""

from __future__ import annotations

import numpy as np

from . import np_oracle

_ROWS = 1 << 12


def _chunk(args):
    # one BLAS thread per process: `cores` then counts exactly the threads used
    # (16 forked workers each spawning a 16-thread BLAS pool oversubscribe the host)
    from threadpoolctl import threadpool_limits
    n, z, c, cw, lo, hi = args
    acc = 0.0
    with threadpool_limits(1):
        for start in range(lo, hi, _ROWS):
            stop = min(start + _ROWS, hi)
            pts = np_oracle.points_block(n, z, start, stop)
            acc += float(np.sum(np.exp(-np.abs(pts @ c - cw))))
    return acc


def cfg5_range_sum(cfg, lo, hi, workers=1):
    """sum_{i in [lo, hi)} exp(-|sum_j c_j (x_ij - w_j)|) on the CPU."""
    z = [pow(cfg.plain_a, j, cfg.plain_n) for j in range(cfg.d)]
    c = np.asarray(cfg.c)
    cw = float(np.dot(c, np.asarray(cfg.w)))
    if workers <= 1:
        return _chunk((cfg.plain_n, z, c, cw, lo, hi))
    import multiprocessing as mp
    bounds = np.linspace(lo, hi, workers + 1).astype(np.int64)
    jobs = [(cfg.plain_n, z, c, cw, int(bounds[k]), int(bounds[k + 1])) for k in range(workers)]
    ctx = mp.get_context("fork")
    with ctx.Pool(workers) as pool:
        return float(sum(pool.map(_chunk, jobs)))
