"""Coefficient generator of arXiv 2512.10059:
region partition, weighted rational Remez exchange, Walsh-table degree search
and the gen pipeline, restated from the reference's regions/remez/polynomial/
linalg/highprec/reference sources in mpmath, with the extremum scan on the
B200 (scan.py).  Test-only cross-check of the native generator (cpp/src/gen): the evaluator
never imports it."""
from .hp import (boys_reference, boys_reference_batch, erf, erfc, gamma_half, precision,  # noqa: F401
                 reference_terms_for, set_working_digits, truncation_bound, upper_gamma_half, working_digits)
from .linalg import jacobi_eigensolve  # noqa: F401
from .poly import (leja_order, newton_interpolate, poly_derivative, poly_eval, poly_trim,  # noqa: F401
                   sturm_root_count)
from .regions import RegionPartition, compute_x0, compute_x1, make_partition, weight_rho_A  # noqa: F401
from .remez import (MT19937_64, FixedNodeCandidate, RationalHP, RemezProblem, RemezResult,  # noqa: F401
                    RemezStatus, WalshResult, golden_section_max, guess_nodes, remez_solve,
                    select_alternating, select_pole_free, solve_fixed_nodes, update_nodes, walsh_search)
