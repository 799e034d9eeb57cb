"""latquad.quad -> paper_2404_08867_b200.quad."""
from paper_2404_08867_b200.quad import *  # noqa: F401,F403
from paper_2404_08867_b200.quad import (QuadratureResult, implr_integrate, mc_integrate,  # noqa: F401
                                        mdilr_integrate, slr_integrate)
from paper_2404_08867_b200.corpus import reference_value  # noqa: F401
