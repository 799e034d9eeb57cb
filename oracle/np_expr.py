"""Literal evaluator of latquad's integrand language (CPU ORACLE, test-only).

The oracle must not share the product's front end (paper_2404_08867_b200.expr
parses into a canonical DAG; the GPU kernels run that DAG).  This module reads
the same source text a second, independent way: it builds a plain syntax tree
(nested tuples, nothing folded, nothing collected) and evaluates that tree
literally over numpy columns.  No canonicalisation happens here, so a bug in
the product's constant splitting, quadratic expansion, angle addition or
like-term collection shows up as a disagreement with this evaluator, while
the reference's own values (tests/golden/parser.json, frozen from
``latquad.exprcore``) pin this evaluator.

Language (the reference's grammar, /root/reference/pkg/src/latquad/
exprcore.py:486-766, restated from its behaviour, plus ``abs``):

* ``+ -`` and ``* /`` left-associative; a ``/`` multiplies by the reciprocal
  of a constant denominator (exprcore.py:569-578) or takes ``c / expr`` as
  ``c * expr^-1``; other denominators are rejected;
* unary ``-`` binds to the operand only, and ``^`` applies to the unary
  result: ``-x[1]^2`` is ``(-x[1])^2`` (exprcore.py:580-592);
* exponents are integer index expressions: ``-k``, ``(iexpr)`` or an atom
  with an optional right-nested ``^`` (exprcore.py:737-757);
* ``pi``, ``e``, ``d``, ``x[iexpr]``, ``exp/sin/cos/abs(expr)``,
  ``sum(i=lo..hi, body)``, ``prod(i=lo..hi, body)`` (empty ranges give 0 and 1);
* index expressions: integers, ``d``, bound indices, ``+ - * /`` (exact
  division only), right-associative ``^`` with a non-negative power, unary
  ``-``, parentheses.

Only well-formed texts need to evaluate here; malformed ones raise
``ValueError`` (the product's error types are pinned separately against the
reference, tests/test_parser_golden.py).
"""

from __future__ import annotations

import math
import re

import numpy as np

_LEX = re.compile(r"""
    (?P<ws>\s+)
  | (?P<num>(?:\d+(?:\.(?!\.)\d*)?|\.\d+)(?:[eE][+-]?\d+)?)
  | (?P<name>[A-Za-z_]\w*)
  | (?P<sym>\.\.|[-+*/^()\[\],=])
""", re.VERBOSE)

_RESERVED = {"d", "x", "pi", "e", "sum", "prod", "exp", "sin", "cos", "abs"}
_UNARY_FN = {"exp": np.exp, "sin": np.sin, "cos": np.cos, "abs": np.abs}


def lex(text):
    out, pos = [], 0
    while pos < len(text):
        m = _LEX.match(text, pos)
        if m is None:
            raise ValueError(f"bad character {text[pos]!r} at {pos}")
        if m.lastgroup != "ws":
            out.append((m.lastgroup, m.group()))
        pos = m.end()
    return out


class _Tree:
    """Token list -> syntax tree.  Node shapes:

    ('lit', float) ('x', ix) ('idx', ix) ('neg', a) ('sum', ((+-1.0, a), ...))
    ('prod', (('*'|'/', a), ...)) ('pow', a, ix) ('fn', name, a)
    ('red', 'sum'|'prod', name, lo_ix, hi_ix, body_tokens)

    where ix is an index-expression tree: ('i', int) ('iname', str)
    ('i+', a, b) ('i-', a, b) ('i*', a, b) ('i/', a, b) ('i^', a, b) ('ineg', a).
    """

    def __init__(self, toks):
        self.toks = toks + [("end", "")]
        self.k = 0

    def look(self):
        return self.toks[self.k][1]

    def next(self):
        t = self.toks[self.k]
        self.k += 1
        return t

    def want(self, s):
        kind, val = self.next()
        if val != s or kind == "end":
            raise ValueError(f"expected {s!r}, got {val!r}")

    # ---- real-valued grammar
    def sum_(self):
        terms = [(1.0, self.prod_())]
        while self.look() in ("+", "-"):
            sign = 1.0 if self.next()[1] == "+" else -1.0
            terms.append((sign, self.prod_()))
        return terms[0][1] if len(terms) == 1 else ("sum", tuple(terms))

    def prod_(self):
        factors = [("*", self.power_())]
        while self.look() in ("*", "/"):
            op = self.next()[1]
            rhs = self.power_()
            if op == "/" and not _is_const(rhs) and not all(_is_const(f) for _, f in factors):
                raise ValueError("non-constant denominator")
            factors.append((op, rhs))
        return factors[0][1] if len(factors) == 1 else ("prod", tuple(factors))

    def power_(self):
        node = self.sign_()
        if self.look() == "^":
            self.next()
            node = ("pow", node, self.exponent_())
        return node

    def sign_(self):
        if self.look() == "-":
            self.next()
            return ("neg", self.atom_())
        return self.atom_()

    def atom_(self):
        kind, val = self.next()
        if kind == "num":
            return ("lit", float(val))
        if val == "(":
            node = self.sum_()
            self.want(")")
            return node
        if kind != "name":
            raise ValueError(f"unexpected {val!r}")
        if val == "pi":
            return ("lit", math.pi)
        if val == "e":
            return ("lit", math.e)
        if val == "x":
            self.want("[")
            ix = self.iadd_()
            self.want("]")
            return ("x", ix)
        if val in _UNARY_FN:
            self.want("(")
            arg = self.sum_()
            self.want(")")
            return ("fn", val, arg)
        if val in ("sum", "prod"):
            self.want("(")
            kind2, name = self.next()
            if kind2 != "name" or name in _RESERVED:
                raise ValueError(f"bad index variable {name!r}")
            self.want("=")
            lo = self.iadd_()
            self.want("..")
            hi = self.iadd_()
            self.want(",")
            # the body is kept as its token span and read once per index value
            # (an empty range never reads it, as in the reference)
            start, depth = self.k, 0
            while True:
                kind3, v3 = self.toks[self.k]
                if kind3 == "end":
                    raise ValueError("unterminated reduction body")
                if v3 in ("(", "["):
                    depth += 1
                elif v3 in (")", "]"):
                    if depth == 0 and v3 == ")":
                        break
                    depth -= 1
                self.k += 1
            body = tuple(self.toks[start:self.k])
            self.want(")")
            return ("red", val, name, lo, hi, body)
        return ("idx", ("iname", val))   # d or a bound index, as a real constant

    # ---- integer index expressions
    def iadd_(self):
        v = self.imul_()
        while self.look() in ("+", "-"):
            op = self.next()[1]
            v = ("i+" if op == "+" else "i-", v, self.imul_())
        return v

    def imul_(self):
        v = self.ipow_()
        while self.look() in ("*", "/"):
            op = self.next()[1]
            v = ("i*" if op == "*" else "i/", v, self.ipow_())
        return v

    def ipow_(self):
        v = self.isign_()
        if self.look() == "^":
            self.next()
            v = ("i^", v, self.ipow_())
        return v

    def isign_(self):
        if self.look() == "-":
            self.next()
            return ("ineg", self.isign_())
        if self.look() == "(":
            self.next()
            v = self.iadd_()
            self.want(")")
            return v
        return self.iatom_()

    def iatom_(self):
        kind, val = self.next()
        if kind == "num" and val.isdigit():
            return ("i", int(val))
        if kind == "name" and val not in _RESERVED - {"d"}:
            return ("iname", val)
        raise ValueError(f"bad index atom {val!r}")

    def exponent_(self):
        # delimited: -k, (iexpr), or atom [^ exponent], so "x^2*y" is (x^2)*y
        if self.look() == "-":
            self.next()
            return ("ineg", self.exponent_())
        if self.look() == "(":
            self.next()
            v = self.iadd_()
            self.want(")")
            return v
        v = self.iatom_()
        if self.look() == "^":
            self.next()
            v = ("i^", v, self.exponent_())
        return v


def _is_const(node):
    """A subtree with no coordinate in it (constant denominators)."""
    tag = node[0]
    if tag == "x":
        return False
    if tag in ("lit", "idx"):
        return True
    if tag in ("neg", "pow"):
        return _is_const(node[1])
    if tag == "fn":
        return _is_const(node[2])
    if tag == "red":
        return _is_const(_body(node[5]))
    return all(_is_const(sub) for _, sub in node[1])   # sum, prod


def _ival(ix, env, d):
    tag = ix[0]
    if tag == "i":
        return ix[1]
    if tag == "iname":
        if ix[1] == "d":
            return d
        if ix[1] not in env:
            raise ValueError(f"unknown index {ix[1]!r}")
        return env[ix[1]]
    if tag == "ineg":
        return -_ival(ix[1], env, d)
    a, b = _ival(ix[1], env, d), _ival(ix[2], env, d)
    if tag == "i+":
        return a + b
    if tag == "i-":
        return a - b
    if tag == "i*":
        return a * b
    if tag == "i/":
        if b == 0 or a % b:
            raise ValueError("inexact index division")
        return a // b
    if b < 0:
        raise ValueError("negative index power")
    return a ** b


def _eval(node, cols, env, d):
    tag = node[0]
    if tag == "lit":
        return node[1]
    if tag == "x":
        i = _ival(node[1], env, d)
        if not 1 <= i <= d:
            raise ValueError(f"x[{i}] outside 1..{d}")
        return cols[i]
    if tag == "idx":
        return float(_ival(node[1], env, d))
    if tag == "neg":
        return -1.0 * _eval(node[1], cols, env, d)
    if tag == "sum":
        acc = None
        for sign, sub in node[1]:
            v = _eval(sub, cols, env, d)
            acc = (v if sign > 0 else -1.0 * v) if acc is None else (acc + v if sign > 0 else acc - v)
        return acc
    if tag == "prod":
        acc = None
        for op, sub in node[1]:
            v = _eval(sub, cols, env, d)
            if op == "/":
                if np.ndim(v) == 0 and v == 0.0:
                    raise ValueError("division by zero")
                v = 1.0 / v   # a/b as a * RN(1/b) (exprcore.py:569-578)
            acc = v if acc is None else acc * v
        return acc
    if tag == "pow":
        b, k = _eval(node[1], cols, env, d), _ival(node[2], env, d)
        if k >= 0:
            return b ** k
        return 1.0 / b if k == -1 else 1.0 / b ** (-k)
    if tag == "fn":
        return _UNARY_FN[node[1]](_eval(node[2], cols, env, d))
    if tag == "red":
        _, which, name, lo, hi, body = node
        acc = 0.0 if which == "sum" else 1.0
        for i in range(_ival(lo, env, d), _ival(hi, env, d) + 1):
            v = _eval(_body(body), cols, {**env, name: i}, d)
            acc = acc + v if which == "sum" else acc * v
        return acc
    raise ValueError(tag)


_CACHE = {}
_BODIES = {}


def _body(toks):
    """Tree of a reduction body from its token span (must be consumed whole)."""
    t = _BODIES.get(toks)
    if t is None:
        p = _Tree(list(toks))
        t = p.sum_()
        if p.toks[p.k][0] != "end":
            raise ValueError("malformed reduction body")
        _BODIES[toks] = t
    return t


def tree(text):
    t = _CACHE.get(text)
    if t is None:
        p = _Tree(lex(text))
        t = p.sum_()
        if p.toks[p.k][0] != "end":
            raise ValueError(f"trailing input {p.look()!r}")
        _CACHE[text] = t
    return t


def evaluate(text, d, cols):
    """Value of the text with x[i] = cols[i] (numpy columns or floats)."""
    return _eval(tree(text), cols, {}, d)
