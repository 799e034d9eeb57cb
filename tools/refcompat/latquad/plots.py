"""latquad.plots: figure rendering (matplotlib) is out of scope."""
from ._oos import _missing

render_suite_figures = _missing("plots.render_suite_figures")
