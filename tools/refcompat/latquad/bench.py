"""latquad.bench -> paper_2404_08867_b200.fits / suites / cli."""
from paper_2404_08867_b200.cli import CSV_COLUMNS, RunRecord  # noqa: F401
from paper_2404_08867_b200.fits import *  # noqa: F401,F403
from paper_2404_08867_b200.fits import DegenerateDataError, FitResult, fit_all, fit_power_law, read_rows  # noqa: F401
from paper_2404_08867_b200.suites import *  # noqa: F401,F403
from paper_2404_08867_b200.suites import SUITES, run_row as _run_row, run_suite, suite_specs  # noqa: F401
