"""Integrand expressions: a small immutable DAG, the reference grammar's
parser, and an adapter that imports the reference's own ``Expr`` objects.

This is the host-side mirror of the part of latquad.exprcore the hot path
consumes (/root/reference/pkg/src/latquad/exprcore.py): ``parse`` accepts the
same source grammar (exprcore.py:488-766, including its quirks: ``-a^k`` is
``(-a)^k`` (exprcore.py:591-603), constant denominators become reciprocal
coefficients (exprcore.py:579-589), ``sum``/``prod`` reductions are expanded at
parse time (exprcore.py:650-673)), plus one extension, ``abs(...)``, which the
BASELINE config-5 integrand needs and the reference lacks (exprcore.py:638).

Unlike the reference we do not canonicalise into a symbolic algebra for
partial summation: the GPU engine never manipulates expressions per node.
Expressions are analysed once (``lower.py``) into either a closed integrand
family with a hand-written kernel, a GPU bytecode program, or a separable
factorisation for MDI-LR.  Light normalisation (flattening, constant folding,
like-term merging) keeps that analysis simple.
"""

from __future__ import annotations

import math

__all__ = [
    "Expr", "ParseError", "UnassignedVariableError",
    "const", "var", "add", "mul", "power", "func",
    "parse", "as_expr", "free_vars", "node_count", "evaluate", "to_text",
]

FUNCS = ("exp", "sin", "cos", "abs")


class ParseError(ValueError):
    """Malformed expression source (mirrors exprcore.ParseError, exprcore.py:72)."""


class UnassignedVariableError(KeyError):
    """Evaluation hit a coordinate with no value (exprcore.py:76)."""


class Expr:
    """Immutable expression node; build with the factories below.

    op: 'const' (val), 'var' (idx, 1-based), 'add' (val = constant,
    terms = ((coef, Expr), ...)), 'mul' (val = coefficient, args = factors),
    'pow' (idx = integer exponent != 0, 1; args = (base,)), or one of
    'exp', 'sin', 'cos', 'abs' (args = (arg,)).
    """

    __slots__ = ("op", "val", "idx", "args", "terms", "_key", "_hash", "_fv", "_fvb")

    def __init__(self, op, val=0.0, idx=0, args=(), terms=()):
        self.op = op
        self.val = float(val) if val != 0.0 else 0.0
        self.idx = int(idx)
        self.args = tuple(args)
        self.terms = tuple(terms)
        if op == "add":
            key = (op, self.val, tuple((c, t._key) for c, t in self.terms))
        else:
            key = (op, self.val, self.idx, tuple(a._key for a in self.args))
        self._key = key
        self._hash = hash(key)
        self._fv = None
        self._fvb = None

    def __hash__(self):
        return self._hash

    def __eq__(self, other):
        return isinstance(other, Expr) and self._hash == other._hash and self._key == other._key

    def __repr__(self):
        return f"Expr<{self.op}:{to_text(self, 60)}>"

    # convenience operators for building test integrands in Python
    def __add__(self, o):
        return add([(1.0, self), (1.0, _lift(o))])

    __radd__ = __add__

    def __sub__(self, o):
        return add([(1.0, self), (-1.0, _lift(o))])

    def __rsub__(self, o):
        return add([(1.0, _lift(o)), (-1.0, self)])

    def __mul__(self, o):
        return mul(1.0, [self, _lift(o)])

    __rmul__ = __mul__

    def __neg__(self):
        return mul(-1.0, [self])

    def __pow__(self, k):
        return power(self, int(k))


def _lift(o):
    return o if isinstance(o, Expr) else const(o)


# ------------------------------------------------------------------ factories

def const(v):
    return Expr("const", float(v))


def var(i):
    if int(i) < 1:
        raise ValueError(f"variable index must be >= 1, got {i}")
    return Expr("var", idx=int(i))


def add(pairs, constant=0.0):
    """Sum of (coef, term) pairs plus a constant; flattens and merges terms."""
    acc = {}
    order = []
    constant = float(constant)
    stack = list(pairs)[::-1]
    while stack:
        coef, t = stack.pop()
        coef = float(coef)
        if coef == 0.0:
            continue
        if t.op == "const":
            constant += coef * t.val
            continue
        if t.op == "add":
            constant += coef * t.val
            stack.extend((coef * c, s) for c, s in reversed(t.terms))
            continue
        if t.op == "mul" and t.val != 1.0:
            coef *= t.val
            t = mul(1.0, t.args)
            if t.op != "mul" or t.val != 1.0:
                stack.append((coef, t))
                continue
        if t in acc:
            acc[t] += coef
        else:
            acc[t] = coef
            order.append(t)
    items = tuple((acc[t], t) for t in order if acc[t] != 0.0)
    if not items:
        return const(constant)
    if len(items) == 1 and constant == 0.0:
        c, t = items[0]
        return t if c == 1.0 else mul(c, [t])
    return Expr("add", constant, terms=items)


def mul(coef, factors):
    """coef * product(factors); flattens products, folds constants and powers."""
    coef = float(coef)
    bases = {}
    order = []
    stack = list(factors)[::-1]
    while stack:
        f = stack.pop()
        if f.op == "const":
            coef *= f.val
            continue
        if f.op == "mul":
            coef *= f.val
            stack.extend(reversed(f.args))
            continue
        base, k = (f.args[0], f.idx) if f.op == "pow" else (f, 1)
        if base in bases:
            bases[base] += k
        else:
            bases[base] = k
            order.append(base)
    if coef == 0.0:
        return const(0.0)
    out = []
    for b in order:
        k = bases[b]
        if k == 0:
            continue
        p = power(b, k)
        if p.op == "const":
            coef *= p.val
        elif p.op == "mul":
            coef *= p.val
            out.extend(p.args)
        else:
            out.append(p)
    if not out:
        return const(coef)
    if len(out) == 1:
        f = out[0]
        if coef == 1.0:
            return f
        if f.op == "add":  # distribute a scalar over a lone sum (exprcore.py:198-202)
            return add([(coef * c, t) for c, t in f.terms], coef * f.val)
    return Expr("mul", coef, args=out)


def power(base, k):
    k = int(k)
    if k == 0:
        return const(1.0)
    if k == 1:
        return base
    if base.op == "const":
        return const(base.val ** k) if k > 0 else const(1.0 / (base.val ** -k))
    if base.op == "pow":
        return power(base.args[0], base.idx * k)
    if base.op == "mul":
        c = base.val ** k if k > 0 else 1.0 / (base.val ** -k)
        return mul(c, [power(f, k) for f in base.args])
    return Expr("pow", idx=k, args=(base,))


def func(name, arg):
    if name not in FUNCS:
        raise ValueError(f"unknown function {name!r}")
    if arg.op == "const":
        v = arg.val
        return const({"exp": math.exp, "sin": math.sin, "cos": math.cos, "abs": abs}[name](v))
    return Expr(name, args=(arg,))


# -------------------------------------------------------------------- queries

def _children(e):
    if e.op == "add":
        return [t for _, t in e.terms]
    return list(e.args)


def topo(e):
    """Nodes reachable from e, children before parents, each once."""
    seen = set()
    out = []
    stack = [(e, False)]
    while stack:
        node, done = stack.pop()
        if done:
            out.append(node)
            continue
        if node in seen:
            continue
        seen.add(node)
        stack.append((node, True))
        for ch in reversed(_children(node)):
            if ch not in seen:
                stack.append((ch, False))
    return out


def node_count(e):
    return len(topo(e))


def free_vars(e):
    """Frozen set of 1-based coordinate indices in e (cached on the node)."""
    if e._fv is None:
        e._fv = frozenset(n.idx for n in topo(e) if n.op == "var")
    return e._fv


def var_bounds(e):
    """(min, max) of free_vars(e), or None without variables (cached on the node)."""
    if e._fvb is None:
        fv = free_vars(e)
        e._fvb = (min(fv), max(fv)) if fv else ()
    return e._fvb or None


def evaluate(e, assignment):
    """Scalar evaluation (host-side helper; the GPU path never calls this)."""
    vals = {}
    for n in topo(e):
        op = n.op
        if op == "const":
            v = n.val
        elif op == "var":
            try:
                v = float(assignment[n.idx])
            except KeyError:
                raise UnassignedVariableError(n.idx) from None
        elif op == "add":
            v = n.val
            for c, t in n.terms:
                v = v + c * vals[t]
        elif op == "mul":
            v = n.val
            for f in n.args:
                v = v * vals[f]
        elif op == "pow":
            b = vals[n.args[0]]
            v = b ** n.idx if n.idx > 0 else 1.0 / (b ** -n.idx)
        else:
            a = vals[n.args[0]]
            v = {"exp": math.exp, "sin": math.sin, "cos": math.cos, "abs": abs}[op](a)
        vals[n] = v
    return float(vals[e])


def to_text(e, maxlen=None):
    def r(n):
        op = n.op
        if op == "const":
            return repr(n.val)
        if op == "var":
            return f"x[{n.idx}]"
        if op == "add":
            parts = [f"{c!r}*{r(t)}" if c != 1.0 else r(t) for c, t in n.terms]
            if n.val != 0.0:
                parts.append(repr(n.val))
            return "(" + " + ".join(parts) + ")"
        if op == "mul":
            body = "*".join(r(f) for f in n.args)
            return body if n.val == 1.0 else f"{n.val!r}*{body}"
        if op == "pow":
            return f"{r(n.args[0])}^({n.idx})"
        return f"{op}({r(n.args[0])})"

    s = r(e)
    if maxlen is not None and len(s) > maxlen:
        s = s[: maxlen - 3] + "..."
    return s


# ------------------------------------------------------- reference Expr import

def as_expr(f):
    """Accept our Expr, or a reference latquad ``Expr`` (duck-typed by its
    kind/value/index/children fields, exprcore.py:80-91), or source text
    with an explicit dimension via ``parse``."""
    if isinstance(f, Expr):
        return f
    if hasattr(f, "kind") and hasattr(f, "children"):
        return _from_reference(f)
    raise TypeError(f"expected an Expr, got {type(f).__name__}")


def _from_reference(root):
    memo = {}
    stack = [(root, False)]
    while stack:
        node, done = stack.pop()
        key = id(node)
        if key in memo:
            continue
        k = node.kind
        if k == "sum":
            kids = [t for t, _ in node.children]
        elif k in ("const", "var"):
            kids = []
        else:
            kids = list(node.children)
        if not done:
            stack.append((node, True))
            stack.extend((c, False) for c in kids if id(c) not in memo)
            continue
        if k == "const":
            out = const(node.value)
        elif k == "var":
            out = var(node.index)
        elif k == "sum":
            out = add([(c, memo[id(t)]) for t, c in node.children], node.value)
        elif k == "prod":
            out = mul(node.value, [memo[id(f)] for f in node.children])
        elif k == "pow":
            out = power(memo[id(node.children[0])], node.index)
        elif k in ("exp", "sin", "cos", "abs"):
            out = func(k, memo[id(node.children[0])])
        else:
            raise TypeError(f"unsupported reference node kind {k!r}")
        memo[key] = out
    return memo[id(root)]


# --------------------------------------------------------------------- parser

def _tokenize(text):
    toks = []
    i, n = 0, len(text)
    while i < n:
        ch = text[i]
        if ch.isspace():
            i += 1
        elif ch.isdigit() or (ch == "." and i + 1 < n and text[i + 1].isdigit()):
            j = i
            while j < n and (text[j].isdigit() or (text[j] == "." and not text.startswith("..", j))):
                j += 1
            if j < n and text[j] in "eE" and text[i:j].count(".") <= 1:
                k = j + 1
                if k < n and text[k] in "+-":
                    k += 1
                if k < n and text[k].isdigit():
                    while k < n and text[k].isdigit():
                        k += 1
                    j = k
            toks.append(("num", text[i:j], i))
            i = j
        elif ch.isalpha() or ch == "_":
            j = i
            while j < n and (text[j].isalnum() or text[j] == "_"):
                j += 1
            toks.append(("name", text[i:j], i))
            i = j
        elif text.startswith("..", i):
            toks.append(("sym", "..", i))
            i += 2
        elif ch in "+-*/^()[],=":
            toks.append(("sym", ch, i))
            i += 1
        else:
            raise ParseError(f"unexpected character {ch!r} at position {i}")
    toks.append(("end", "", n))
    return toks


_RESERVED = ("d", "x", "pi", "e", "sum", "prod") + FUNCS


class _Parser:
    def __init__(self, toks, d, env):
        self.toks, self.pos, self.d, self.env = toks, 0, d, env

    def peek(self):
        return self.toks[self.pos]

    def take(self, want=None):
        tok = self.toks[self.pos]
        if want is not None and tok[1] != want:
            raise ParseError(f"expected {want!r} at position {tok[2]}, found {tok[1]!r}")
        self.pos += 1
        return tok

    # real-valued grammar
    def expr(self):
        pairs = [(1.0, self.term())]
        while self.peek()[1] in ("+", "-"):
            sign = 1.0 if self.take()[1] == "+" else -1.0
            pairs.append((sign, self.term()))
        return add(pairs) if len(pairs) > 1 else pairs[0][1]

    def term(self):
        node = self.factor()
        while self.peek()[1] in ("*", "/"):
            op = self.take()[1]
            at = self.peek()[2]
            rhs = self.factor()
            if op == "*":
                node = mul(1.0, [node, rhs])
            elif rhs.op == "const":
                if rhs.val == 0.0:
                    raise ParseError(f"division by zero at position {at}")
                node = mul(1.0 / rhs.val, [node])
            elif node.op == "const":
                node = mul(node.val, [power(rhs, -1)])
            else:
                raise ParseError(f"non-constant denominator at position {at}")
        return node

    def factor(self):
        node = self.unary()
        if self.peek()[1] == "^":
            self.take("^")
            node = power(node, self.ipower())
        return node

    def unary(self):
        if self.peek()[1] == "-":
            self.take("-")
            return mul(-1.0, [self.base()])
        return self.base()

    def base(self):
        kind, val, at = self.peek()
        if kind == "num":
            self.take()
            try:
                return const(float(val))
            except ValueError:
                raise ParseError(f"bad numeric literal {val!r} at position {at}") from None
        if val == "(":
            self.take("(")
            node = self.expr()
            self.take(")")
            return node
        if kind == "name":
            self.take()
            if val == "pi":
                return const(math.pi)
            if val == "e":
                return const(math.e)
            if val == "x":
                self.take("[")
                i = self.iexpr()
                self.take("]")
                if not 1 <= i <= self.d:
                    raise ParseError(f"coordinate x[{i}] outside 1..{self.d} at position {at}")
                return var(i)
            if val in FUNCS:
                self.take("(")
                arg = self.expr()
                self.take(")")
                return func(val, arg)
            if val in ("sum", "prod"):
                return self.reduction(val)
            if val in self.env:
                return const(float(self.env[val]))
            if val == "d":
                return const(float(self.d))
            raise ParseError(f"unknown identifier {val!r} at position {at}")
        raise ParseError(f"unexpected token {val!r} at position {at}")

    def reduction(self, which):
        self.take("(")
        kind, name, at = self.take()
        if kind != "name" or name in _RESERVED:
            raise ParseError(f"bad index variable {name!r} at position {at}")
        self.take("=")
        lo = self.iexpr()
        self.take("..")
        hi = self.iexpr()
        self.take(",")
        start = self.pos
        depth = 0
        while True:
            k, v, p = self.toks[self.pos]
            if k == "end":
                raise ParseError(f"unterminated body at position {p}")
            if v in ("(", "["):
                depth += 1
            elif v in (")", "]"):
                if depth == 0 and v == ")":
                    break
                depth -= 1
            self.pos += 1
        end = self.pos
        self.take(")")
        parts = []
        for i in range(lo, hi + 1):
            sub = _Parser(self.toks, self.d, {**self.env, name: i})
            sub.pos = start
            parts.append(sub.expr())
            if sub.pos != end:
                raise ParseError(f"malformed {which} body at position {at}")
        if not parts:
            return const(0.0 if which == "sum" else 1.0)
        return add([(1.0, p) for p in parts]) if which == "sum" else mul(1.0, parts)

    # integer index arithmetic
    def iexpr(self):
        v = self.iterm()
        while self.peek()[1] in ("+", "-"):
            op = self.take()[1]
            r = self.iterm()
            v = v + r if op == "+" else v - r
        return v

    def iterm(self):
        v = self.ifactor()
        while self.peek()[1] in ("*", "/"):
            op = self.take()[1]
            at = self.peek()[2]
            r = self.ifactor()
            if op == "*":
                v *= r
            else:
                if r == 0 or v % r != 0:
                    raise ParseError(f"non-integer division in index expression at {at}")
                v //= r
        return v

    def ifactor(self):
        v = self.iunary()
        if self.peek()[1] == "^":
            self.take("^")
            k = self.ifactor()
            if k < 0:
                raise ParseError("negative power in index expression")
            v = v ** k
        return v

    def iunary(self):
        if self.peek()[1] == "-":
            self.take("-")
            return -self.iunary()
        if self.peek()[1] == "(":
            self.take("(")
            v = self.iexpr()
            self.take(")")
            return v
        return self.iatom()

    def iatom(self):
        kind, val, at = self.take()
        if kind == "num":
            if "." in val or "e" in val or "E" in val:
                raise ParseError(f"non-integer literal {val!r} in index expression at {at}")
            return int(val)
        if kind == "name":
            if val == "d":
                return self.d
            if val in self.env:
                return self.env[val]
            raise ParseError(f"unknown index identifier {val!r} at position {at}")
        raise ParseError(f"unexpected token {val!r} in index expression at {at}")

    def ipower(self):
        if self.peek()[1] == "-":
            self.take("-")
            return -self.ipower()
        if self.peek()[1] == "(":
            self.take("(")
            v = self.iexpr()
            self.take(")")
            return v
        v = self.iatom()
        if self.peek()[1] == "^":
            self.take("^")
            k = self.ipower()
            if k < 0:
                raise ParseError("negative power in index expression")
            v = v ** k
        return v


def parse(text, d):
    """Parse source text into an Expr; ``d`` bounds x[i] (exprcore.py:759-766)."""
    p = _Parser(_tokenize(text), int(d), {})
    node = p.expr()
    if p.peek()[0] != "end":
        _, val, at = p.peek()
        raise ParseError(f"trailing input {val!r} at position {at}")
    return node
