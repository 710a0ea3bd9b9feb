"""refine_symmetric (refine.py:409-438) on the GPU against the reference's own
runs (tests/golden/symmetric_ref.*, made by tests/golden/make_golden.py from
the unmodified reference): dd mode (the reference's precision pair) and FP64
mode on the same Hermitian inputs, plus the NotSymmetric rejection."""
import numpy as np
import pytest
import torch

from paper_2203_10879_b200 import NotSymmetric, RefineConfig, RefineStatus, refine_symmetric, verify_pair

pytestmark = pytest.mark.gpu

U_HP = 2.0 ** -106
U64 = 2.0 ** -53


def ref_diag(arr, k):
    return (arr["trh_%d" % k] + arr["trl_%d" % k]) + 1j * (arr["tih_%d" % k] + arr["til_%d" % k])


def test_symmetric_dd_matches_reference(golden):
    meta, arr = golden("symmetric_ref")
    for c in meta["cases"]:
        k, n = c["k"], c["n"]
        a = arr["a_%d" % k]
        pair, rep = refine_symmetric(a, RefineConfig(seed=c["seed"]))
        assert rep.status.value == c["status"], (c, rep.status)
        assert abs(rep.iterations - c["iterations"]) <= 1, (c, rep.iterations)
        assert rep.hp_matmul_count == 2 + 4 * rep.iterations - (1 if rep.skip_fired else 0)
        assert len(rep.residual_history) == rep.iterations + 1
        # same eigenvalue order (random line of the same seed) and values to dd accuracy
        t = pair.t.to_numpy_cells()
        d = np.diag(t[0]) + np.diag(t[1])
        dref = ref_diag(arr, k).real
        assert np.abs(d - dref).max() <= 1e-28 * np.abs(dref).max(), (c, np.abs(d - dref).max())
        assert not np.any(t[2]) and not np.any(t[3])  # real T (refine.py:435-436)
        v = verify_pair(a, pair)
        norm_a = np.linalg.norm(a)
        assert v.ortho_residual <= 1e-28 and v.tri_residual <= 10 * n * U_HP * norm_a


def test_symmetric_fp64_matches_reference_order_and_values(golden):
    meta, arr = golden("symmetric_ref")
    for c in meta["cases"]:
        k, n = c["k"], c["n"]
        a = arr["a_%d" % k]
        pair, rep = refine_symmetric(a, RefineConfig(precision="fp64", tol_factor=10.0 / n, max_iters=10,
                                                     seed=c["seed"]))
        assert rep.status is RefineStatus.CONVERGED, (c, rep.status, rep.detail)
        t = pair.t.cpu().numpy()
        dref = ref_diag(arr, k).real
        assert np.abs(np.diag(t).real - dref).max() <= 50 * U64 * np.abs(dref).max()
        assert not np.any(t.imag)
        off = t - np.diag(np.diag(t))
        assert np.linalg.norm(off) <= 10 * n * U64 * np.linalg.norm(a)
        v = verify_pair(a, pair, precision="fp64")
        assert v.ortho_residual <= 10 * n * U64 and v.tri_residual <= 10 * n * U64 * np.linalg.norm(a)


def test_symmetric_rejects_non_hermitian(golden):
    meta, arr = golden("symmetric_ref")
    for precision in ("dd", "fp64"):
        with pytest.raises(NotSymmetric):
            refine_symmetric(arr["a_nonsym"], RefineConfig(precision=precision))


def test_symmetric_real_input_large():
    """A real symmetric matrix at n = 700 in FP64 mode (the real-A product path):
    converges, diagonal T equal to the sorted eigenvalues (numpy eigvalsh)."""
    rng = np.random.default_rng(11)
    x = rng.standard_normal((700, 700))
    a = (x + x.T) / 2
    pair, rep = refine_symmetric(a, RefineConfig(precision="fp64", tol_factor=10.0 / 700, max_iters=10))
    assert rep.status is RefineStatus.CONVERGED, rep
    d = np.sort(np.diag(pair.t.cpu().numpy()).real)
    ev = np.linalg.eigvalsh(a)
    assert np.abs(d - ev).max() <= 1e-12 * np.abs(ev).max()

