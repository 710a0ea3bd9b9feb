"""refine_mixed (refine.py:383-406) on the GPU against the reference's own runs
(tests/golden/mixed_ref.*): the GPU lp Schur front end (eigenpairs in the
random-line order + QR) must reproduce the reference's eigenvalue order, and
the refined pair its diagonal to dd accuracy (dd mode) / FP64 accuracy."""
import numpy as np
import pytest

from paper_2203_10879_b200 import RefineConfig, RefineStatus, refine_mixed, verify_pair

pytestmark = pytest.mark.gpu

U_HP = 2.0 ** -106
U64 = 2.0 ** -53


def ref_diag(arr, k):
    return (arr["trh_%d" % k] + arr["trl_%d" % k]) + 1j * (arr["tih_%d" % k] + arr["til_%d" % k])


def test_mixed_dd_matches_reference(golden):
    meta, arr = golden("mixed_ref")
    for c in meta["cases"]:
        k, n = c["k"], c["n"]
        a = arr["a_%d" % k]
        pair, rep = refine_mixed(a, RefineConfig(seed=c["seed"]))
        assert rep.status.value == c["status"], (c, rep.status)
        assert abs(rep.iterations - c["iterations"]) <= 1, (c, rep.iterations)
        assert rep.hp_matmul_count == 2 + 4 * rep.iterations - (1 if rep.skip_fired else 0)
        t = pair.t.to_numpy_cells()
        d = (np.diag(t[0]) + np.diag(t[1])) + 1j * (np.diag(t[2]) + np.diag(t[3]))
        dref = ref_diag(arr, k)
        assert np.abs(d - dref).max() <= 1e-28 * np.abs(dref).max(), (c, np.abs(d - dref).max())
        v = verify_pair(a, pair)
        assert v.ortho_residual <= 1e-28 and v.tri_residual <= 10 * n * U_HP * np.linalg.norm(a)


def test_mixed_fp64_matches_reference_order(golden):
    meta, arr = golden("mixed_ref")
    for c in meta["cases"]:
        k, n = c["k"], c["n"]
        a = arr["a_%d" % k]
        pair, rep = refine_mixed(a, RefineConfig(precision="fp64", tol_factor=10.0 / n, max_iters=10,
                                                 seed=c["seed"]))
        assert rep.status is RefineStatus.CONVERGED, (c, rep.status, rep.detail)
        d = np.diag(pair.t.cpu().numpy())
        dref = ref_diag(arr, k)
        assert np.abs(d - dref).max() <= 100 * U64 * np.abs(dref).max(), (c, np.abs(d - dref).max())
        v = verify_pair(a, pair, precision="fp64")
        assert v.tri_residual <= 10 * n * U64 * np.linalg.norm(a) and v.ortho_residual <= 10 * n * U64


def test_mixed_fp64_n1024_from_scratch():
    """n = 1024 complex Gaussian from scratch in FP64 mode (front end on the
    GPU, no CPU Schur): converges within the iteration budget, and the result
    passes the FP64 verify_pair at the stop rule."""
    from paper_2203_10879_b200 import inputs
    a = inputs.gaussian_complex(1024, 3)
    pair, rep = refine_mixed(a, RefineConfig(precision="fp64", tol_factor=10.0 / 1024, max_iters=10))
    assert rep.status is RefineStatus.CONVERGED and rep.iterations <= 6, rep
    v = verify_pair(a, pair, precision="fp64")
    assert v.tri_residual <= 10 * 1024 * U64 * np.linalg.norm(a) and v.ortho_residual <= 10 * 1024 * U64
