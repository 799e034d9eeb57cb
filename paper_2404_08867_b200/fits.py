"""Power-law cost models over benchmark CSV rows, so timings of the GPU
engine drop into the reference's scaling analysis (the caller side of the
path; behaviour of latquad.bench.fit_power_law /
fit_all, /root/reference/pkg/src/latquad/bench.py:254-340).

Every model is ``t = c * N^k * v^p`` with a fixed power k of the points per
axis N and a fitted exponent p on one sweep variable v; p and c come from a
straight line through (log v, log t - k log N), R^2 is taken on the seconds
themselves.  Host statistics on a few rows -- nothing here is on the GPU.
"""

from __future__ import annotations

import csv
import math
from dataclasses import dataclass
from pathlib import Path

import numpy as np

__all__ = ["MODELS", "FitResult", "DegenerateDataError", "read_rows", "fit_power_law", "fit_all"]

# model name -> (fixed power k of N, sweep variable carrying the fitted exponent)
_SHAPES = {"N^p": (0, "N"), "N*d^q": (1, "d"), "N^2*d^q": (2, "d")}
MODELS = tuple(_SHAPES)

# CSV column -> type of its non-empty cells (RunRecord schema, cli.CSV_COLUMNS)
_TYPED = {"d": int, "n": int, "a": int, "seed": int,
          "value": float, "reference": float, "rel_error": float, "seconds": float}


class DegenerateDataError(ValueError):
    """The rows leave a model nothing to fit (no sweep, constant timings)."""


@dataclass
class FitResult:
    model: str
    coeff: float
    exponent: float
    r_squared: float
    count: int

    def formatted(self):
        k, var = _SHAPES[self.model]
        base = {0: "", 1: "N*", 2: "N^2*"}[k]
        return (f"t = {self.coeff:.4g}*{base}{var}^{self.exponent:.4g}  "
                f"(R2={self.r_squared:.4f}, {self.count} rows)")


def read_rows(path):
    """Rows of a RunRecord CSV as dicts, typed per _TYPED (empty cells -> None)."""
    with open(path, newline="") as fh:
        return [{k: (_TYPED[k](v) if v else None) if k in _TYPED else v for k, v in raw.items()}
                for raw in csv.DictReader(fh)]


def _samples(rows):
    """(N, d, t) arrays of the rows that ran ('ok' or no status) and carry seconds."""
    if isinstance(rows, (str, Path)):
        rows = read_rows(rows)

    def field(row, key):
        return row.get(key) if isinstance(row, dict) else getattr(row, key, None)

    kept = [(field(r, "a"), field(r, "d"), field(r, "seconds")) for r in rows
            if field(r, "status") in (None, "", "ok") and field(r, "seconds") is not None]
    if any(N is None or d is None for N, d, _ in kept):
        raise ValueError("fit rows need both a (points per axis) and d columns")
    arr = np.asarray(kept, dtype=float).reshape(-1, 3)
    return arr[:, 0], arr[:, 1], arr[:, 2]


def _line(x, y):
    """Least-squares slope and intercept of y against x (closed form)."""
    xm, ym = x.mean(), y.mean()
    dx = x - xm
    slope = float(np.dot(dx, y - ym) / np.dot(dx, dx))
    return slope, float(ym - slope * xm)


def fit_power_law(rows, model):
    """Fit one model; raises ValueError on unusable rows and
    DegenerateDataError when the model's sweep variable or the timings do not vary."""
    if model not in _SHAPES:
        raise ValueError(f"unknown model {model!r}; expected one of {MODELS}")
    N, d, t = _samples(rows)
    if t.size < 4:
        raise ValueError(f"need at least 4 usable rows, got {t.size}")
    if (t <= 0).any():
        raise ValueError("fit requires positive wall seconds in every row")
    k, var = _SHAPES[model]
    v = N if var == "N" else d
    x = np.log(v)
    if x.max() == x.min():
        raise DegenerateDataError(f"model {model} needs variation in its sweep variable")
    p, log_c = _line(x, np.log(t) - k * np.log(N))
    c = math.exp(log_c)
    spread = float(((t - t.mean()) ** 2).sum())
    if spread == 0.0:
        raise DegenerateDataError("constant timings: R^2 undefined")
    resid = t - c * N ** k * v ** p
    return FitResult(model, c, p, 1.0 - float((resid ** 2).sum()) / spread, int(t.size))


def fit_all(rows):
    """All models that admit a fit, best R^2 first."""
    fitted = []
    for model in MODELS:
        try:
            fitted.append(fit_power_law(rows, model))
        except DegenerateDataError:
            pass
    if not fitted:
        raise DegenerateDataError("no model family admits a fit on this data")
    return sorted(fitted, key=lambda r: -r.r_squared)
