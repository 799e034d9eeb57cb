"""latquad.exprcore -> paper_2404_08867_b200.expr (factories under the
reference's names; the symbolic level operations are out of scope)."""

from paper_2404_08867_b200.expr import (Expr, ParseError, UnassignedVariableError, const, free_vars,  # noqa: F401
                                        node_count, parse, to_text, var)
from paper_2404_08867_b200.mdi import DEFAULT_NODE_BUDGET, BudgetExceededError  # noqa: F401
from paper_2404_08867_b200.expr import add as _add, func as _func, mul as _mul, power as _power
from paper_2404_08867_b200.expr import evaluate as eval  # noqa: A001,F401
from paper_2404_08867_b200.engine import eval_array  # noqa: F401

from ._oos import bind, normalize, partial_sum, substitute  # noqa: F401


def make_sum(pairs, constant=0.0):
    return _add([(c, t) for t, c in pairs], constant)


def make_prod(coef, factors):
    return _mul(coef, factors)


def make_pow(base, k):
    return _power(base, k)


def exp_of(x):
    return _func("exp", x)


def sin_of(x):
    return _func("sin", x)


def cos_of(x):
    return _func("cos", x)
