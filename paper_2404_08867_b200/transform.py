"""Lattice -> tensor-grid axis counts and the improved rule's midpoint grids
(drop-in for latquad.transform's value-path API,
/root/reference/pkg/src/latquad/transform.py:48-83, 169-178).

The exact rational forward transform, general-z grid validation and the
transformed integrand (transform.py:86-166, 181-242) never feed the value
 and are out of scope.
"""

from __future__ import annotations

import math

import numpy as np

__all__ = ["AxisGridSet", "axis_counts", "midpoint_grids"]


class AxisGridSet:
    """Per-axis node tuples with their counts and the source rule
    (transform.py:48-73).  Midpoint grids keep their nodes implicit --
    RN((t + 0.5) / n_i) is regenerated on the GPU -- and materialise the
    tuples only when ``nodes`` is read."""

    __slots__ = ("counts", "n", "z", "_nodes", "midpoint", "_total")

    def __init__(self, nodes, counts, n, z, midpoint=False):
        counts = tuple(int(c) for c in counts)
        if nodes is not None:
            nodes = tuple(tuple(float(v) for v in nd) for nd in nodes)
            if len(nodes) != len(counts):
                raise ValueError("nodes/counts length mismatch")
            for ax, (nd, ct) in enumerate(zip(nodes, counts)):
                if len(nd) != ct:
                    raise ValueError(f"axis {ax + 1} has {len(nd)} nodes, expected {ct}")
        self.counts = counts
        self.n = n
        self.z = z
        self._nodes = nodes
        self.midpoint = midpoint
        self._total = None

    @property
    def nodes(self):
        if self._nodes is None:
            self._nodes = tuple(tuple((t + 0.5) / ct for t in range(ct)) for ct in self.counts)
        return self._nodes

    @property
    def d(self):
        return len(self.counts)

    @property
    def total(self):
        if self._total is None:
            self._total = math.prod(self.counts)
        return self._total

    def node_arrays(self):
        return [np.asarray(nd, dtype=float) for nd in self.nodes]

    def __eq__(self, other):
        return (isinstance(other, AxisGridSet) and self.counts == other.counts
                and self.n == other.n and self.z == other.z and self.nodes == other.nodes)

    def __hash__(self):
        return hash((self.counts, self.n, self.z))

    def __repr__(self):
        return f"AxisGridSet(d={self.d}, counts={self.counts[:6]}{'...' if self.d > 6 else ''})"


def axis_counts(rule):
    """(n_1, ..., n_d): lcm(z_i, z_{i+1}) // min(z_i, z_{i+1}) for i < d and
    ceil(n / z_d), in exact integer arithmetic on the unreduced z
    (transform.py:76-83).  Korobov rules use the closed form n_i = a."""
    z, n = rule.z, rule.n
    a = getattr(rule, "_korobov_a", None)
    if a is not None and rule.d > 1:
        return (a,) * (rule.d - 1) + (-(-n // z[-1]),)
    out = []
    for i in range(rule.d - 1):
        out.append(math.lcm(z[i], z[i + 1]) // min(z[i], z[i + 1]))
    out.append(-(-n // z[-1]))
    return tuple(out)


def midpoint_grids(rule):
    """Open grids: nodes (t + 1/2)/n_i with the rule's axis counts (transform.py:169-178).
    Immutable, so one grid set is kept per (immutable) rule object."""
    g = rule.__dict__.get("_midpoint_grids")
    if g is None:
        g = AxisGridSet(None, axis_counts(rule), rule.n, rule.z, midpoint=True)
        object.__setattr__(rule, "_midpoint_grids", g)
    return g
