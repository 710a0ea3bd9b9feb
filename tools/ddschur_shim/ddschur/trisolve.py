"""ddschur.trisolve: the GPU solver with the reference's counters."""
from paper_2203_10879_b200.errors import NonFiniteError, SeparationError  # noqa: F401
from paper_2203_10879_b200.trisolve import (TriEqProblem, TriEqSolution, reset_stats, solve_block,  # noqa: F401
                                            solve_scalar, stats)

from . import reference_module


def __getattr__(name):  # phi_estimate, solve_sylvester_tri: off the hot path
    if name.startswith("__"):
        raise AttributeError(name)
    return getattr(reference_module("trisolve"), name)
