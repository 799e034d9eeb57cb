"""latquad.transform -> paper_2404_08867_b200.transform (validation path out of scope)."""
from paper_2404_08867_b200.transform import AxisGridSet, axis_counts, midpoint_grids  # noqa: F401

from ._oos import (NonCartesianStructureError, TransformedIntegrand, build_axis_grids,  # noqa: F401
                   forward_transform, grid_completion, inverse_substitution, make_transformed_integrand)
