"""Power-law cost fits over RunRecord rows, so GPU timings drop into the
reference's scaling analysis (/root/reference/pkg/src/latquad/bench.py:254-340,
SURVEY.md §8(f) item 4).  Host-side statistics on timing rows, not a sum."""

from __future__ import annotations

import csv
import math
from dataclasses import dataclass
from pathlib import Path

import numpy as np

__all__ = ["MODELS", "FitResult", "DegenerateDataError", "read_rows", "fit_power_law", "fit_all"]

MODELS = ("N^p", "N*d^q", "N^2*d^q")


class DegenerateDataError(ValueError):
    """Fit data carries no usable variation (constant inputs or outputs)."""


@dataclass
class FitResult:
    model: str
    coeff: float
    exponent: float
    r_squared: float
    count: int

    def formatted(self):
        shape = {"N^p": "N^{e}", "N*d^q": "N*d^{e}", "N^2*d^q": "N^2*d^{e}"}[self.model]
        return f"t = {self.coeff:.4g}*{shape.format(e=f'{self.exponent:.4g}')}  (R2={self.r_squared:.4f}, {self.count} rows)"


def read_rows(path):
    """A RunRecord CSV back into typed dicts (empty cells -> None)."""
    out = []
    with open(path, newline="") as fh:
        for raw in csv.DictReader(fh):
            row = dict(raw)
            for k in ("d", "n", "a", "seed"):
                row[k] = int(raw[k]) if raw.get(k) else None
            for k in ("value", "reference", "rel_error", "seconds"):
                row[k] = float(raw[k]) if raw.get(k) else None
            out.append(row)
    return out


def _columns(rows):
    if isinstance(rows, (str, Path)):
        rows = read_rows(rows)
    N, d, t = [], [], []
    for row in rows:
        get = row.get if isinstance(row, dict) else (lambda k, r=row: getattr(r, k, None))
        if get("status") not in (None, "", "ok") or get("seconds") is None:
            continue
        N.append(get("a"))
        d.append(get("d"))
        t.append(get("seconds"))
    if any(v is None for v in N) or any(v is None for v in d):
        raise ValueError("fit rows need both a (points per axis) and d columns")
    return np.asarray(N, float), np.asarray(d, float), np.asarray(t, float)


def fit_power_law(rows, model):
    """Least squares in log space (slope = exponent); R^2 in linear space."""
    if model not in MODELS:
        raise ValueError(f"unknown model {model!r}; expected one of {MODELS}")
    N, d, t = _columns(rows)
    if len(t) < 4:
        raise ValueError(f"need at least 4 usable rows, got {len(t)}")
    if np.any(t <= 0):
        raise ValueError("fit requires positive wall seconds in every row")
    lt = np.log(t)
    if model == "N^p":
        x, y = np.log(N), lt
    elif model == "N*d^q":
        x, y = np.log(d), lt - np.log(N)
    else:
        x, y = np.log(d), lt - 2.0 * np.log(N)
    if np.ptp(x) == 0.0:
        raise DegenerateDataError(f"model {model} needs variation in its sweep variable")
    slope, icpt = np.polyfit(x, y, 1)
    coeff = math.exp(icpt)
    pred = coeff * (N ** slope if model == "N^p" else (N if model == "N*d^q" else N * N) * d ** slope)
    ss = float(np.sum((t - t.mean()) ** 2))
    if ss == 0.0:
        raise DegenerateDataError("constant timings: R^2 undefined")
    return FitResult(model, coeff, float(slope), 1.0 - float(np.sum((t - pred) ** 2)) / ss, len(t))


def fit_all(rows):
    """Every model that admits a fit, best R^2 first."""
    res = []
    for m in MODELS:
        try:
            res.append(fit_power_law(rows, m))
        except DegenerateDataError:
            continue
    if not res:
        raise DegenerateDataError("no model family admits a fit on this data")
    return sorted(res, key=lambda r: r.r_squared, reverse=True)
