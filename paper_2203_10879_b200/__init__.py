"""B200-native Schur refinement (arXiv 2203.10879): a drop-in for the
reference package's `refine_template` hot path.  Public names follow the
reference's `ddschur/__init__.py`."""
from .errors import NonFiniteError, NormTooLarge, NotSymmetric, SeparationError
from .matmul import counters, matmul_hp, matmul_lp, reset_counters
from .matrix import ZPlanar
from .refine import (
    U_FP64,
    U_HP,
    OrthoStrategy,
    RefineConfig,
    RefineReport,
    RefineStatus,
    SchurPair,
    refine_template,
    VerifyResiduals,
    verify_pair,
)
from .trisolve import TriEqProblem, TriEqSolution, reset_stats, solve_block, solve_scalar, stats
from .ddmatrix import DDMatrix, DDScalar, frobenius_norm, precision_convert, stril_extract
from .orthogonal import merged_update, newton_schulz_step
from .continuation import refine_continuation
from .symmetric import order_by_random_line, refine_symmetric
from .mixed import refine_mixed
from .matrix import DDPlanar

__version__ = "0.1.0"
__all__ = [
    "NonFiniteError", "NormTooLarge", "NotSymmetric", "SeparationError", "counters", "matmul_hp",
    "matmul_lp", "reset_counters", "ZPlanar", "U_FP64", "U_HP", "OrthoStrategy", "RefineConfig",
    "RefineReport", "RefineStatus", "SchurPair", "refine_template", "verify_pair", "VerifyResiduals", "TriEqProblem",
    "TriEqSolution", "solve_block", "refine_continuation", "DDPlanar", "refine_symmetric",
    "order_by_random_line", "refine_mixed", "solve_scalar", "stats", "reset_stats", "DDMatrix", "DDScalar",
    "frobenius_norm", "precision_convert", "stril_extract", "merged_update", "newton_schulz_step",
]
