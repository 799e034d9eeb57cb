"""latquad.lattice -> paper_2404_08867_b200.lattice + quality."""
from paper_2404_08867_b200.lattice import *  # noqa: F401,F403
from paper_2404_08867_b200.lattice import (LatticeRule, fibonacci_rule, iter_point_blocks, korobov_vector,  # noqa: F401
                                           lattice_points, points_block)
from paper_2404_08867_b200.quality import *  # noqa: F401,F403
from paper_2404_08867_b200.quality import (QualityWarning, WeightModel, bernoulli_poly, cbc_construct,  # noqa: F401
                                           korobov_search, p_alpha, shift_avg_wce_sq)
