"""latquad.bench -> paper_2404_08867_b200.fits / suites / cli."""
from paper_2404_08867_b200.cli import RunRecord  # noqa: F401
from paper_2404_08867_b200.fits import *  # noqa: F401,F403
from paper_2404_08867_b200.fits import DegenerateDataError, FitResult, fit_all, fit_power_law  # noqa: F401
from paper_2404_08867_b200.suites import *  # noqa: F401,F403
from paper_2404_08867_b200.suites import run_suite, suite_specs  # noqa: F401
