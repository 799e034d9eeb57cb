"""B200-native rank-1 lattice sums and MDI-LR (arXiv 2404.08867), a drop-in
for the hot path of the reference package ``latquad``.

Same names, argument meaning and errors as latquad's value-path API
(/root/reference/pkg/src/latquad/__init__.py:4-94, the subset listed in
SURVEY.md §8(b)); every sum over points, grid nodes or clusters runs in the
sm_100a library ``liblq.so`` (include/lq.h).
"""

from .expr import Expr, ParseError, UnassignedVariableError, as_expr, free_vars, node_count, parse, to_text
from .expr import evaluate as eval  # noqa: A001 -- the reference's contract name (exprcore.py:404)
from .engine import eval_array
from .lattice import LatticeRule, fibonacci_rule, iter_point_blocks, korobov_vector, lattice_points, points_block
from .transform import AxisGridSet, axis_counts, midpoint_grids
from .mdi import (DEFAULT_NODE_BUDGET, DIRECT_CAP, BudgetExceededError, GridCapError, MdiConfig,
                  MdiReport, direct_tensor_sum, mdi_lr, mdi_sum)
from .quad import QuadratureResult, implr_integrate, mc_integrate, mdilr_integrate, slr_integrate
from .quality import (QualityWarning, WeightModel, bernoulli_poly, cbc_construct, korobov_search, p_alpha,
                      shift_avg_wce_sq)
from .corpus import CorpusEntry, all_ids, corpus_expr, entries, get, reference_value
from .fits import DegenerateDataError, FitResult, fit_all, fit_power_law
from .cli import RunRecord, cli_main
from .suites import run_suite, suite_specs

__version__ = "0.1.0"

__all__ = [
    "Expr", "ParseError", "UnassignedVariableError", "as_expr", "free_vars", "node_count", "parse", "to_text",
    "eval", "eval_array",
    "LatticeRule", "fibonacci_rule", "iter_point_blocks", "korobov_vector", "lattice_points", "points_block",
    "AxisGridSet", "axis_counts", "midpoint_grids",
    "DEFAULT_NODE_BUDGET", "DIRECT_CAP", "BudgetExceededError", "GridCapError", "MdiConfig",
    "MdiReport", "direct_tensor_sum", "mdi_lr", "mdi_sum",
    "QuadratureResult", "implr_integrate", "mc_integrate", "mdilr_integrate", "slr_integrate",
    "QualityWarning", "WeightModel", "bernoulli_poly", "cbc_construct", "korobov_search", "p_alpha",
    "shift_avg_wce_sq",
    "CorpusEntry", "all_ids", "corpus_expr", "entries", "get", "reference_value",
    "DegenerateDataError", "FitResult", "fit_all", "fit_power_law", "RunRecord", "cli_main",
    "run_suite", "suite_specs",
    "__version__",
]
