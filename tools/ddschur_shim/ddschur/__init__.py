"""Import shim: `import ddschur` resolves to the B200 drop-in for the hot path.

For a maintainer with a GPU and the reference source, to run the reference's
OWN hot-path tests against paper_2203_10879_b200 in dd mode:

    DDSCHUR_REF_SRC=/path/to/reference/pkg/src \
    PYTHONPATH=tools/ddschur_shim:. python -m pytest /path/to/reference/pkg/tests/test_refine.py -k "..."

(tools/run_reference_tests.sh lists the hot-path cases).  Hot-path names come
from paper_2203_10879_b200 (GPU, no CPU fallback); host utilities outside the
hot path (generators, Matrix Market, CLI, the binary64 Schur front end,
qr_retract, phi_estimate) are taken from the REAL reference found at
$DDSCHUR_REF_SRC.  Results come back as host DDMatrix containers, like the
reference's.  This shim is test tooling, not product code.
"""
import importlib.util
import os
import sys

_REF = os.environ.get("DDSCHUR_REF_SRC")


def reference_module(name):
    """The unmodified reference module ddschur.<name> (loaded under another name)."""
    if not _REF:
        raise ImportError("set DDSCHUR_REF_SRC to the reference's pkg/src for ddschur.%s" % name)
    key = "_ddschur_ref." + name
    if key in sys.modules:
        return sys.modules[key]
    if "_ddschur_ref" not in sys.modules:
        spec = importlib.util.spec_from_file_location("_ddschur_ref", os.path.join(_REF, "ddschur", "__init__.py"),
                                                      submodule_search_locations=[os.path.join(_REF, "ddschur")])
        pkg = importlib.util.module_from_spec(spec)
        sys.modules["_ddschur_ref"] = pkg
        spec.loader.exec_module(pkg)
    return importlib.import_module(key)


from paper_2203_10879_b200 import (  # noqa: E402,F401
    DDMatrix, NonFiniteError, NormTooLarge, NotSymmetric, OrthoStrategy, RefineReport, RefineStatus,
    SeparationError, TriEqProblem, TriEqSolution, U_HP, VerifyResiduals, counters, frobenius_norm, matmul_hp,
    matmul_lp, merged_update, newton_schulz_step, precision_convert, reset_counters, solve_block, solve_scalar,
    stril_extract, verify_pair)
from .refine import RefineConfig, refine_mixed, refine_symmetric, refine_template  # noqa: E402,F401
