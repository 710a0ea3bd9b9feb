#!/bin/bash
# Run the reference's own hot-path tests against the B200 drop-in (dd mode).
# Needs a B200 AND the reference source: DDSCHUR_REF_SRC=<reference>/pkg/src.
# (The restated versions of these cases run in tests/test_gpu_boundary.py.)
set -e
: "${DDSCHUR_REF_SRC:?set DDSCHUR_REF_SRC to the reference's pkg/src}"
T=$(dirname "$DDSCHUR_REF_SRC")/tests
export PYTHONPATH="$(dirname "$0")/ddschur_shim:$(cd "$(dirname "$0")/.." && pwd):$PYTHONPATH"
python -m pytest -q "$T/test_refine.py" -k "exact_candidate or quadratic_residual or repeated_eigenvalue or contraction or shape_and_validation or config_validation or nonfinite or verify_exact or verify_identity"
python -m pytest -q "$T/test_acceptance.py" -k "quadratic_convergence_order or orthogonalization_step_contract or triangular_solvers_match_dense_oracle"
python -m pytest -q "$T/test_trisolve.py" -k "invocation_counters"
