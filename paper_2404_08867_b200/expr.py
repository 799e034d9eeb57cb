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
import weakref
import re

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

    __slots__ = ("op", "val", "idx", "args", "terms", "_key", "_hash", "_fv", "_fvb", "__weakref__")

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

    # latquad's field names (exprcore.py:80-91), read-only views of this node
    # for callers that inspect a parsed expression
    @property
    def kind(self):
        return {"add": "sum", "mul": "prod"}.get(self.op, self.op)

    @property
    def value(self):
        return self.val

    @property
    def index(self):
        return self.idx

    @property
    def children(self):
        if self.op == "add":
            return tuple((t, c) for c, t in self.terms)
        return self.args


def _lift(o):
    return o if isinstance(o, Expr) else const(o)


# ------------------------------------------------------------------ factories

# One live object per distinct node (the reference hash-conses its DAG the
# same way, exprcore.py:94-106, and callers may rely on `parse(t) is parse(t)`)
_INTERN = weakref.WeakValueDictionary()


def _node(op, val=0.0, idx=0, args=(), terms=()):
    e = Expr(op, val, idx, args, terms)
    return _INTERN.setdefault(e._key, e)


def const(v):
    return _node("const", float(v))


def var(i):
    if int(i) < 1:
        raise ValueError(f"variable index must be >= 1, got {i}")
    return _node("var", idx=int(i))


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
    return _node("add", constant, terms=items)


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
    return _node("mul", coef, args=out)


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
    return _node("pow", idx=k, args=(base,))


def func(name, arg):
    if name not in FUNCS:
        raise ValueError(f"unknown function {name!r}")
    if arg.op == "const":
        v = arg.val
        return const({"exp": math.exp, "sin": math.sin, "cos": math.cos, "abs": abs}[name](v))
    return _node(name, args=(arg,))


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


def _num(v):
    """Integers without a fraction part, anything else as repr (exprcore.py:778-781)."""
    return str(int(v)) if v == int(v) and abs(v) < 1e15 else repr(v)


def to_text(e, maxlen=None):
    """Readable rendering for diagnostics, in latquad's conventions
    (exprcore.py:771-818): variables as x1, powers b^k, a product's
    coefficient in front, sums joined by + / -, parentheses by precedence
    (0 sum, 1 product, 2 atom).  Not meant to be parsed back."""
    def atom(n):
        return n.op not in ("add", "mul")

    def r(n, prec):
        op = n.op
        if op == "const":
            return _num(n.val)
        if op == "var":
            return f"x{n.idx}"
        if op == "pow":
            b = r(n.args[0], 2)
            if not atom(n.args[0]):
                b = f"({b})"
            return f"{b}^{n.idx}" if n.idx != -1 else f"{b}^-1"
        if op == "mul":
            body = "*".join(r(f, 2) if f.op != "add" else f"({r(f, 0)})" for f in n.args)
            if n.val != 1.0:
                body = f"{_num(n.val)}*{body}"
            return f"({body})" if prec > 1 else body
        if op == "add":
            parts = []
            for c, t in n.terms:
                rt = r(t, 1)
                parts.append(rt if c == 1.0 else f"-{rt}" if c == -1.0 else f"{_num(c)}*{rt}")
            if n.val != 0.0 or not parts:
                parts.append(_num(n.val))
            body = " + ".join(parts).replace("+ -", "- ")
            return f"({body})" if prec > 0 else body
        return f"{op}({r(n.args[0], 0)})"

    s = r(e, 0)
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

_TOKEN_RE = re.compile(r"""
    (?P<ws>\s+)
  | (?P<num>(?:\d|\.(?=\d))(?:\d|\.(?!\.))*)
  | (?P<name>[^\W\d]\w*)
  | (?P<sym>\.\.|[-+*/^()\[\],=])
""", re.VERBOSE)
_EXPONENT_RE = re.compile(r"[eE][+-]?\d+")


def _scan(text):
    """Token list [(kind, text, position)] ending with ('end', '', len).  A
    numeric literal runs over digits and single dots ('..' is the range
    separator) and takes a decimal exponent only when it has at most one dot."""
    out = []
    pos = 0
    while pos < len(text):
        m = _TOKEN_RE.match(text, pos)
        if m is None:
            raise ParseError(f"character {text[pos]!r} at {pos} is not part of the grammar")
        kind = m.lastgroup
        end = m.end()
        if kind == "num" and m.group().count(".") <= 1:
            ex = _EXPONENT_RE.match(text, end)
            if ex is not None:
                end = ex.end()
        if kind != "ws":
            out.append((kind, text[pos:end], pos))
        pos = end
    out.append(("end", "", len(text)))
    return out


# Binary operators of the real-valued grammar: token -> binding power.  Every
# operator is left-associative; '^' is not here: an exponent is an integer
# index expression applied once to a unary operand (see _Reader.power_operand).
_BINARY = {"+": 10, "-": 10, "*": 20, "/": 20}
_RESERVED = frozenset(("d", "x", "pi", "e", "sum", "prod") + FUNCS)
_CONSTANTS = {"pi": math.pi, "e": math.e}


class _Reader:
    """Reads the token list into a small syntax tree once (precedence
    climbing over _BINARY); sum/prod bodies are stored as trees and expanded
    by _Builder per index value.  A body that does not read cleanly is kept
    as its error and raised only if its range is non-empty, the way an
    expansion-time parse would behave."""

    def __init__(self, toks):
        self.toks = toks
        self.i = 0

    def at(self):
        return self.toks[self.i]

    def advance(self):
        tok = self.toks[self.i]
        self.i += 1
        return tok

    def expect(self, text):
        kind, got, pos = self.toks[self.i]
        if kind != "sym" or got != text:
            raise ParseError(f"{text!r} expected at {pos} (got {got or 'end of input'!r})")
        self.i += 1

    def expression(self, floor=0):
        lhs = self.power_operand()
        while True:
            _, op, pos = self.at()
            bp = _BINARY.get(op)
            if bp is None or bp <= floor or self.at()[0] != "sym":
                return lhs
            self.advance()
            lhs = ("bin", op, lhs, self.expression(bp), pos)

    def power_operand(self):
        node = self.unary()
        if self.at()[1] == "^" and self.at()[0] == "sym":
            self.advance()
            node = ("pow", node, self.exponent())
        return node

    def unary(self):
        if self.at()[1] == "-" and self.at()[0] == "sym":
            self.advance()
            return ("neg", self.primary())      # -a^k reads as (-a)^k
        return self.primary()

    def primary(self):
        kind, text, pos = self.advance()
        if kind == "num":
            try:
                return ("num", float(text))
            except ValueError:
                raise ParseError(f"malformed number {text!r} at {pos}") from None
        if kind == "sym" and text == "(":
            node = self.expression()
            self.expect(")")
            return node
        if kind != "name":
            raise ParseError(f"{text or 'end of input'!r} at {pos} cannot start an operand")
        if text == "x":
            self.expect("[")
            idx = self.index_expression()
            self.expect("]")
            return ("x", idx, pos)
        if text in FUNCS:
            self.expect("(")
            arg = self.expression()
            self.expect(")")
            return ("call", text, arg)
        if text in ("sum", "prod"):
            return self.reduction(text, pos)
        return ("name", text, pos)

    def reduction(self, which, pos):
        self.expect("(")
        kind, var, vpos = self.advance()
        if kind != "name" or var in _RESERVED:
            raise ParseError(f"{var!r} at {vpos} cannot be a {which} index")
        self.expect("=")
        lo = self.index_expression()
        self.expect("..")
        hi = self.index_expression()
        self.expect(",")
        first = self.i
        depth = 0
        while True:                       # the body runs to the ')' that closes the call
            kind, text, tpos = self.at()
            if kind == "end":
                raise ParseError(f"{which} body starting at {self.toks[first][2]} is never closed")
            if text in "([" and kind == "sym":
                depth += 1
            elif text in ")]" and kind == "sym":
                if depth == 0 and text == ")":
                    break
                depth -= 1
            self.i += 1
        last = self.i
        self.advance()
        sub = _Reader(self.toks[first:last] + [("end", "", self.toks[last][2])])
        try:
            body = sub.expression()
            if sub.at()[0] != "end":
                raise ParseError(f"{which} body at {pos} does not end where its call closes")
        except ParseError as exc:
            body = exc
        return ("red", which, var, lo, hi, body)

    # integer index expressions: + - * / (exact), ^ (right-assoc, k >= 0), unary -
    def index_expression(self):
        v = self.index_term()
        while self.at()[1] in ("+", "-") and self.at()[0] == "sym":
            op = self.advance()[1]
            v = ("ibin", op, v, self.index_term(), None)
        return v

    def index_term(self):
        v = self.index_factor()
        while self.at()[1] in ("*", "/") and self.at()[0] == "sym":
            op = self.advance()[1]
            pos = self.at()[2]
            v = ("ibin", op, v, self.index_factor(), pos)
        return v

    def index_factor(self):
        v = self.index_unary()
        if self.at()[1] == "^" and self.at()[0] == "sym":
            self.advance()
            v = ("ipow", v, self.index_factor())
        return v

    def index_unary(self):
        kind, text, _ = self.at()
        if kind == "sym" and text == "-":
            self.advance()
            return ("ineg", self.index_unary())
        if kind == "sym" and text == "(":
            self.advance()
            v = self.index_expression()
            self.expect(")")
            return v
        return self.index_atom()

    def index_atom(self):
        kind, text, pos = self.advance()
        if kind == "num":
            if not text.isdigit():
                raise ParseError(f"index expressions take integers, got {text!r} at {pos}")
            return ("inum", int(text))
        if kind == "name":
            return ("iname", text, pos)
        raise ParseError(f"{text or 'end of input'!r} at {pos} is not an index operand")

    def exponent(self):
        """An exponent is delimited: '-' exponent | '(' index expression ')' |
        atom ['^' exponent], so 'x^2*y' is (x^2)*y."""
        kind, text, _ = self.at()
        if kind == "sym" and text == "-":
            self.advance()
            return ("ineg", self.exponent())
        if kind == "sym" and text == "(":
            self.advance()
            v = self.index_expression()
            self.expect(")")
            return v
        v = self.index_atom()
        if self.at()[1] == "^" and self.at()[0] == "sym":
            self.advance()
            v = ("ipow", v, self.exponent())
        return v


class _Builder:
    """Syntax tree -> Expr under an environment of index values."""

    def __init__(self, d):
        self.d = d

    def index(self, t, env):
        tag = t[0]
        if tag == "inum":
            return t[1]
        if tag == "iname":
            if t[1] == "d":
                return self.d
            if t[1] in env:
                return env[t[1]]
            raise ParseError(f"{t[1]!r} at {t[2]} is not an index in scope")
        if tag == "ineg":
            return -self.index(t[1], env)
        if tag == "ipow":
            b, k = self.index(t[1], env), self.index(t[2], env)
            if k < 0:
                raise ParseError(f"index power {b}^{k} has a negative exponent")
            return b ** k
        op, a, b = t[1], self.index(t[2], env), self.index(t[3], env)
        if op == "+":
            return a + b
        if op == "-":
            return a - b
        if op == "*":
            return a * b
        if b == 0 or a % b:
            raise ParseError(f"{a}/{b} at {t[4]} is not an exact integer division")
        return a // b

    def real(self, t, env):
        tag = t[0]
        if tag == "num":
            return const(t[1])
        if tag == "name":
            name = t[1]
            if name in _CONSTANTS:
                return const(_CONSTANTS[name])
            if name in env:
                return const(float(env[name]))
            if name == "d":
                return const(float(self.d))
            raise ParseError(f"unknown name {name!r} at {t[2]}")
        if tag == "x":
            j = self.index(t[1], env)
            if not 1 <= j <= self.d:
                raise ParseError(f"x[{j}] at {t[2]} is outside the coordinates 1..{self.d}")
            return var(j)
        if tag == "call":
            return func(t[1], self.real(t[2], env))
        if tag == "neg":
            return mul(-1.0, [self.real(t[1], env)])
        if tag == "pow":
            return power(self.real(t[1], env), self.index(t[2], env))
        if tag == "red":
            return self.reduction(t, env)
        return self.chain(t, env)

    def chain(self, t, env):
        """A left-leaning run of one precedence level, folded iteratively (long
        sums of thousands of terms stay off the Python stack): '+'/'-' runs
        build one n-ary sum, '*'/'/' runs fold left to right."""
        group = "+-" if t[1] in "+-" else "*/"
        spine = []
        node = t
        while node[0] == "bin" and node[1] in group:
            spine.append(node)
            node = node[2]
        acc = self.real(node, env)
        if group == "+-":
            pairs = [(1.0, acc)]
            for n in reversed(spine):
                pairs.append((1.0 if n[1] == "+" else -1.0, self.real(n[3], env)))
            return add(pairs)
        for n in reversed(spine):
            rhs = self.real(n[3], env)
            if n[1] == "*":
                acc = mul(1.0, [acc, rhs])
            elif rhs.op == "const":
                # by a constant: its reciprocal as the coefficient
                if rhs.val == 0.0:
                    raise ParseError(f"division by zero at {n[4]}")
                acc = mul(1.0 / rhs.val, [acc])
            elif acc.op == "const":
                # a constant over an expression: its -1 power
                acc = mul(acc.val, [power(rhs, -1)])
            else:
                raise ParseError(f"quotient at {n[4]} has a non-constant numerator and denominator")
        return acc

    def reduction(self, t, env):
        _, which, name, lo, hi, body = t
        lo, hi = self.index(lo, env), self.index(hi, env)
        if hi < lo:
            return const(0.0 if which == "sum" else 1.0)
        if isinstance(body, ParseError):
            raise body
        parts = [self.real(body, {**env, name: i}) for i in range(lo, hi + 1)]
        return add([(1.0, p) for p in parts]) if which == "sum" else mul(1.0, parts)


def parse(text, d):
    """Source text -> Expr over coordinates x[1..d] (the grammar of
    exprcore.parse, exprcore.py:486-766, plus abs(...))."""
    reader = _Reader(_scan(text))
    tree = reader.expression()
    kind, tok, pos = reader.at()
    if kind != "end":
        raise ParseError(f"unexpected {tok!r} at {pos} after a complete expression")
    return _Builder(int(d)).real(tree, {})
