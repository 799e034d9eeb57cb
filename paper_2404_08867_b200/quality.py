"""Lattice quality measures and constructions on the GPU (drop-in for the
rule-selection half of latquad.lattice, /root/reference/pkg/src/latquad/
lattice.py:140-311, "the step before" the lattice sum).

Every sum over points and candidates runs in liblq.so (``lq_bprod_sum``,
``lq_cbc_construct``, ``lq_korobov_values``); the host keeps the reference's
validation, weights, anchors and the strict-improvement tie rule.
"""

from __future__ import annotations

import ctypes as C
import math
import warnings
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .lattice import LatticeRule, korobov_vector

__all__ = ["WeightModel", "QualityWarning", "bernoulli_poly", "p_alpha", "shift_avg_wce_sq",
           "cbc_construct", "korobov_search"]


class QualityWarning(UserWarning):
    """A quality measure was evaluated for a rule with gcd(z_j, n) != 1 (lattice.py:46-47)."""


@dataclass(frozen=True)
class WeightModel:
    """Product weights gamma_j with the anchor constant beta (lattice.py:184-215)."""

    gamma: tuple
    beta: float = 0.0

    def __post_init__(self):
        object.__setattr__(self, "gamma", tuple(float(g) for g in self.gamma))
        object.__setattr__(self, "beta", float(self.beta))
        if any(g <= 0.0 for g in self.gamma):
            raise ValueError("product weights must be positive")

    @classmethod
    def unanchored(cls, gamma):
        return cls(tuple(gamma), 0.0)

    @classmethod
    def anchored(cls, gamma, c=1.0):
        return cls(tuple(gamma), c * c - c + 1.0 / 3.0)

    @classmethod
    def default(cls, d):
        return cls(tuple(1.0 / (j * j) for j in range(1, d + 1)), 0.0)

    def prefix(self, k):
        return WeightModel(self.gamma[:k], self.beta)


def bernoulli_poly(x, alpha):
    """B_2 or B_4 on [0, 1) (lattice.py:140-149); host helper for user data."""
    x = np.asarray(x, dtype=float)
    if alpha == 2:
        t = x - 0.5
        return t * t - 1.0 / 12.0
    if alpha == 4:
        return ((x - 2.0) * x + 1.0) * x * x - 1.0 / 30.0
    raise ValueError(f"alpha must be 2 or 4, got {alpha}")


def _warn_grid_type(rule, measure):
    if rule.is_grid_type:
        warnings.warn(f"{measure} assumes gcd(z_j, n) = 1; rule n={rule.n} z={rule.z} is grid-type "
                      "and the measure does not certify its accuracy", QualityWarning, stacklevel=3)


def _bprod(rule, alpha, g, beta):
    if rule.n > 2**53:
        raise OverflowError(f"cannot sweep an n={rule.n} rule")
    g = np.ascontiguousarray(g, dtype=np.float64)
    out = C.c_double()
    N.check(N.lib().lq_bprod_sum(N.ctx(), alpha, rule.d, rule.n, N.as_ptr(rule.z_reduced_array()),
                                 N.as_ptr(g), float(beta), 0, rule.n, C.byref(out)))
    return out.value


def p_alpha(rule, alpha=2):
    """Figure of merit P_alpha by the Bernoulli closed form (lattice.py:167-181)."""
    if alpha not in (2, 4):
        raise ValueError(f"alpha must be 2 or 4, got {alpha}")
    _warn_grid_type(rule, "p_alpha")
    sign = 1.0 if (alpha // 2) % 2 == 1 else -1.0
    coef = sign * (2.0 * math.pi) ** alpha / math.factorial(alpha)
    total = _bprod(rule, alpha, [coef] * rule.d, 0.0)
    return total / rule.n - 1.0


def _weights_for(d, weights):
    w = weights if weights is not None else WeightModel.default(d)
    if len(w.gamma) < d:
        raise ValueError(f"need {d} weights, got {len(w.gamma)}")
    return w.gamma[:d], w.beta


def shift_avg_wce_sq(rule, weights=None):
    """Squared shift-averaged worst-case error (lattice.py:225-245)."""
    gamma, beta = _weights_for(rule.d, weights)
    anchor = float(np.prod(1.0 + np.asarray(gamma) * beta))
    total = _bprod(rule, 2, gamma, beta)
    return total / rule.n - anchor


def _improves(val, best):
    return val < best - 1e-9 * abs(best)      # lattice.py:248-252


def _coprime_candidates(n):
    return [c for c in range(1, n) if math.gcd(c, n) == 1]


def cbc_construct(n, d, weights=None):
    """Component-by-component rule (lattice.py:259-289), every candidate sweep on the GPU."""
    if n < 2:
        raise ValueError(f"component-by-component search needs n >= 2, got {n}")
    if d < 1:
        raise ValueError(f"dimension must be positive, got {d}")
    w = weights if weights is not None else WeightModel.default(d)
    if len(w.gamma) < d:
        raise ValueError(f"need {d} weights, got {len(w.gamma)}")
    cands = np.asarray(_coprime_candidates(n), dtype=np.int64)
    gamma = np.ascontiguousarray(w.gamma[:d], dtype=np.float64)
    z = np.zeros(d, dtype=np.int64)
    N.check(N.lib().lq_cbc_construct(N.ctx(), n, d, N.as_ptr(gamma), float(w.beta), N.as_ptr(cands),
                                     len(cands), N.as_ptr(z)))
    return LatticeRule(n, tuple(int(v) for v in z))


def korobov_search(n, d, weights=None, criterion="wce"):
    """Best Korobov rule over the coprime a (lattice.py:292-311), ties to the smallest a."""
    if n < 2:
        raise ValueError(f"Korobov search needs n >= 2, got {n}")
    if criterion not in ("wce", "p2"):
        raise ValueError(f"criterion must be 'wce' or 'p2', got {criterion!r}")
    cands = np.asarray(_coprime_candidates(n), dtype=np.int64)
    if criterion == "wce":
        gamma, beta = _weights_for(d, weights)
        anchor = float(np.prod(1.0 + np.asarray(gamma) * beta))
    else:
        coef = (2.0 * math.pi) ** 2 / 2.0
        gamma, beta, anchor = (coef,) * d, 0.0, 1.0
    g = np.ascontiguousarray(gamma, dtype=np.float64)
    sums = np.zeros(len(cands))
    N.check(N.lib().lq_korobov_values(N.ctx(), n, d, N.as_ptr(g), float(beta), N.as_ptr(cands), len(cands),
                                      N.as_ptr(sums)))
    best_a, best_val = None, math.inf
    for a, s in zip(cands.tolist(), sums.tolist()):
        val = s / n - anchor
        if best_a is None or _improves(val, best_val):
            best_a, best_val = a, val
    return korobov_vector(best_a, n, d)
