"""Named integrands with closed-form references, so runs can be requested by
id exactly as latquad's CLI and suites do (/root/reference/pkg/src/latquad/
corpus.py:89-151).  Host-side metadata only; the sums run on the GPU.

Each entry: (id, expression text in d, minimum d, reference integral over
[0,1]^d as a function of d).
"""

from __future__ import annotations

import cmath
import math
from dataclasses import dataclass

from .expr import parse

__all__ = ["CorpusEntry", "all_ids", "corpus_expr", "entries", "get", "reference_value", "text_of"]


def _one(d):
    return 1.0


def _gauss_1d():
    from scipy.special import erf
    return math.sqrt(math.pi / 2.0) * float(erf(1.0 / math.sqrt(2.0)))


def _erfi_factor():
    from scipy.special import erfi
    return math.sqrt(math.pi) / 2.0 * float(erfi(1.0))


def _erf_factor():
    from scipy.special import erf
    return math.sqrt(math.pi) / 2.0 * float(erf(1.0))


def _fresnel_w():
    from scipy.special import fresnel
    s, c = fresnel(math.sqrt(2.0 / math.pi))
    return math.sqrt(math.pi / 2.0) * complex(float(c), float(s))


_RAT = (math.atan(0.4 / 0.9) + math.atan(0.6 / 0.9)) / 0.9
_COSLIN = (cmath.exp(2.0j) - 1.0) / 2.0j

_TABLE = {
    "expxy": ("x[2]*exp(x[1]*x[2])/(e-2)", 2, _one),
    "sinsq": ("sin(2*pi + sum(i=1..d, x[i]^2))", 1, lambda d: (_fresnel_w() ** d).imag),
    "expsum": ("exp(sum(i=1..d, x[i])) / (e-1)^d", 1, _one),
    "gaussian": ("0.3989422804014327*exp(-sum(i=1..d, x[i]^2)/2)", 1,
                 lambda d: (1.0 / math.sqrt(2.0 * math.pi)) * _gauss_1d() ** d),
    "expalt": ("exp(sum(i=1..d, (-1)^(i+1)*x[i]))", 1,
               lambda d: (math.e - 1.0) ** ((d + 1) // 2) * (1.0 - 1.0 / math.e) ** (d // 2)),
    "ratprod": ("prod(i=1..d, 1/(0.81 + (x[i]-0.6)^2))", 1, lambda d: _RAT ** d),
    "coslin": ("cos(2*pi + sum(i=1..d, 2*x[i]))", 1, lambda d: (_COSLIN ** d).real),
    "expsq": ("exp(sum(i=1..d, (-1)^(i+1)*x[i]^2))", 1,
              lambda d: _erfi_factor() ** ((d + 1) // 2) * _erf_factor() ** (d // 2)),
    "invpow": ("(1 + sum(i=1..d, x[i]))^(-(d+1))", 1, lambda d: 1.0 / math.factorial(d + 1)),
    "one": ("1", 1, _one),
}


# benchmark families each integrand appears in (the reference's suites, bench.py)
_SUITES = {
    "expxy": ("test1",), "sinsq": ("test1", "test2"), "expsum": ("test2",),
    "gaussian": ("test3", "test5", "test6", "test7"), "expalt": ("test4", "test7"),
    "ratprod": ("test4", "test5", "test6", "test7"), "coslin": ("test5", "test6", "test7"),
    "expsq": ("test7",), "invpow": ("test7",), "one": (),
}


@dataclass(frozen=True)
class CorpusEntry:
    """One named integrand (corpus.py:68-86): id, source text in d, exact
    integral as a function of d, the suites it appears in, minimum d."""

    id: str
    text: str
    reference: object
    suites: tuple
    min_d: int = 1

    def expr(self, d):
        if d < self.min_d:
            raise ValueError(f"{self.id} needs d >= {self.min_d}, got {d}")
        return parse(self.text, d)

    def ref(self, d):
        return float(self.reference(d))


_ENTRIES = {k: CorpusEntry(k, text, fn, _SUITES[k], min_d) for k, (text, min_d, fn) in _TABLE.items()}


def entries():
    return list(_ENTRIES.values())


def get(name):
    try:
        return _ENTRIES[name]
    except KeyError:
        raise KeyError(f"unknown integrand {name!r}; known: {', '.join(_TABLE)}") from None


def all_ids():
    return list(_TABLE)


def text_of(name):
    try:
        return _TABLE[name][0]
    except KeyError:
        raise KeyError(f"unknown integrand {name!r}; known: {', '.join(_TABLE)}") from None


def corpus_expr(name, d):
    text, min_d, _ = _TABLE[name] if name in _TABLE else (text_of(name), 1, None)
    if d < min_d:
        raise ValueError(f"{name} needs d >= {min_d}, got {d}")
    return parse(text, d)


def reference_value(name, d):
    """Exact integral of the named integrand over [0,1]^d, or None."""
    entry = _TABLE.get(name)
    return None if entry is None else float(entry[2](d))
