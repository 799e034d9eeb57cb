"""latquad.mdi -> paper_2404_08867_b200.mdi."""
from paper_2404_08867_b200.mdi import *  # noqa: F401,F403
from paper_2404_08867_b200.mdi import (DEFAULT_NODE_BUDGET, DIRECT_CAP, BudgetExceededError, GridCapError,  # noqa: F401
                                       MdiConfig, MdiReport, direct_tensor_sum, mdi_lr, mdi_sum)
