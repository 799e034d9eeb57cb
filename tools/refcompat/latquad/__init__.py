"""Compatibility shim: the import name ``latquad`` resolving to this repo's
package (paper_2404_08867_b200), so that the reference's own test suite can be
run unmodified against the GPU implementation (tools/run_reference_tests.py).
Names that exist only in the reference's symbolic engine or transform
validation path (out of scope, SURVEY §2 / DESIGN §8) raise NotImplementedError
when called."""

from paper_2404_08867_b200 import *  # noqa: F401,F403
from paper_2404_08867_b200 import __all__, __version__  # noqa: F401

from . import bench, cli, corpus, exprcore, lattice, mdi, plots, quad, transform  # noqa: F401,E402

from ._oos import (NonCartesianStructureError, TransformedIntegrand, bind, build_axis_grids,  # noqa: F401,E402
                   forward_transform, grid_completion, inverse_substitution, make_transformed_integrand,
                   partial_sum, substitute)
