"""Seeded synthetic workloads of BASELINE.json ``configs``.

Every array here feeds both the CPU oracle and the CUDA path, so the two see
bit-identical inputs.  The reference measures on no public dataset; these
seeded Genz-style integrands with the stated shapes stand in.

Draw order per config (``np.random.default_rng(k)`` for config k, the PCG64
generator latquad itself uses, /root/reference/pkg/src/latquad/quad.py:84):
``a = rng.integers(2, n)`` (plain-sum lattices only) -> ``c = rng.uniform(0, 1, d)``
-> ``w = rng.uniform(0, 1, d)`` (configs 3-5) -> ``u = rng.uniform()`` (config 2);
then ``c *= S / c.sum()``.

Integrand source text uses ``repr(float)`` literals, which the reference
tokenizer reads back exactly (/root/reference/pkg/src/latquad/exprcore.py:496-509).
Config 5 uses ``abs``, which the reference grammar lacks
(exprcore.py:638 raises ParseError); our parser accepts it as an extension.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

__all__ = ["SynthConfig", "make_config", "CONFIG_IDS", "family_text"]

CONFIG_IDS = (1, 2, 3, 4, 5)


@dataclass(frozen=True)
class SynthConfig:
    """One BASELINE.json config: integrand parameters plus its two lattices."""

    cid: int
    d: int
    family: str                 # expsum_lin | osc | gauss_peak | prod_peak | exp_abs_lin
    text: str                   # expression source (reference grammar, + abs for cfg5)
    plain_n: int = None         # plain lattice sum: n (prime), Korobov a (seeded)
    plain_a: int = None
    mdi_a: int = None           # MDI-LR: a = N, n = N^d  (cfg1: seeded a, n = 1009)
    mdi_n: int = None
    c: tuple = field(default=(), repr=False)
    w: tuple = field(default=(), repr=False)
    u: float = None
    exact: float = None         # closed-form integral over [0,1]^d where known

    def plain_z(self):
        """z_reduced = a^(j-1) mod n, the plain-sum generating vector
        (/root/reference/pkg/src/latquad/lattice.py:76-78, 132-137)."""
        return tuple(pow(self.plain_a, j, self.plain_n) for j in range(self.d))


def _rescale(c, total):
    c = np.asarray(c, dtype=float)
    return c * (total / c.sum())


def family_text(family, d, c=(), w=(), u=None):
    """Expression text for a family with the given parameters."""
    if family == "expsum_lin":
        return "exp(sum(i=1..d, x[i])/d)"
    if family == "osc":
        terms = " + ".join(f"{float(cj)!r}*x[{j + 1}]" for j, cj in enumerate(c))
        return f"cos(2*pi*{float(u)!r} + {terms})"
    if family == "gauss_peak":
        terms = " + ".join(f"{float(cj) ** 2!r}*(x[{j + 1}]-{float(wj)!r})^2"
                           for j, (cj, wj) in enumerate(zip(c, w)))
        return f"exp(-({terms}))"
    if family == "prod_peak":
        facs = " * ".join(f"(1/({float(cj) ** -2!r} + (x[{j + 1}]-{float(wj)!r})^2))"
                          for j, (cj, wj) in enumerate(zip(c, w)))
        return facs
    if family == "exp_abs_lin":
        terms = " + ".join(f"{float(cj)!r}*(x[{j + 1}]-{float(wj)!r})"
                           for j, (cj, wj) in enumerate(zip(c, w)))
        return f"exp(-abs({terms}))"
    raise ValueError(f"unknown family {family!r}")


def make_config(cid):
    """Build config ``cid`` (1..5) of BASELINE.json deterministically."""
    rng = np.random.default_rng(cid)
    if cid == 1:
        d, n = 8, 1009
        a = int(rng.integers(2, n))
        exact = (d * (np.exp(1.0 / d) - 1.0)) ** d
        return SynthConfig(1, d, "expsum_lin", family_text("expsum_lin", d),
                           plain_n=n, plain_a=a, mdi_a=a, mdi_n=n, exact=float(exact))
    if cid == 2:
        d, n, N = 100, 10007, 64
        a = int(rng.integers(2, n))
        c = _rescale(rng.uniform(0.0, 1.0, d), 9.0)
        u = float(rng.uniform())
        return SynthConfig(2, d, "osc", family_text("osc", d, c=c, u=u),
                           plain_n=n, plain_a=a, mdi_a=N, mdi_n=N ** d,
                           c=tuple(map(float, c)), u=u)
    if cid == 3:
        d, n = 300, 1_000_003
        a = int(rng.integers(2, n))
        c = _rescale(rng.uniform(0.0, 1.0, d), 7.0)
        w = rng.uniform(0.0, 1.0, d)
        return SynthConfig(3, d, "gauss_peak", family_text("gauss_peak", d, c=c, w=w),
                           plain_n=n, plain_a=a, c=tuple(map(float, c)), w=tuple(map(float, w)))
    if cid == 4:
        d, N = 500, 256
        c = _rescale(rng.uniform(0.0, 1.0, d), 25.0)
        w = rng.uniform(0.0, 1.0, d)
        return SynthConfig(4, d, "prod_peak", family_text("prod_peak", d, c=c, w=w),
                           mdi_a=N, mdi_n=N ** d, c=tuple(map(float, c)), w=tuple(map(float, w)))
    if cid == 5:
        d, n, N = 1000, 2**31 - 1, 512
        a = int(rng.integers(2, n))
        c = _rescale(rng.uniform(0.0, 1.0, d), 10.0)
        w = rng.uniform(0.0, 1.0, d)
        return SynthConfig(5, d, "exp_abs_lin", family_text("exp_abs_lin", d, c=c, w=w),
                           plain_n=n, plain_a=a, mdi_a=N, mdi_n=N ** d,
                           c=tuple(map(float, c)), w=tuple(map(float, w)))
    raise ValueError(f"config id must be 1..5, got {cid}")
