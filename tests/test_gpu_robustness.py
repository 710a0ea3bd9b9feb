"""Robustness cases the r1 verdict asked for (items 9 / weak 2, 11):

  * graded inputs for the Ozaki-II products (rows / columns scaled by
    2^+-20): per-row and per-column power-of-two scaling makes a diagonally
    graded product D1 A B D2 as accurate, entry by entry relative to
    (|A||B|)_ij, as an ungraded one; grading INSIDE a row (columns of A
    scaled) keeps the normwise bound — the limit the reference's own Ozaki
    path documents (pkg/README.md:58-63) — checked against the dd oracle;
  * restore_full_sigma=True (orthogonal.py:197-200) through the whole FP64
    refinement against the restatement with the same flag;
  * exact clip-count parity of the complex64 solve (tensor-core far updates)
    at n = 2048 against the C restatement (trisolve.py:141-144,192-195).
"""
import numpy as np
import pytest
import torch

from oracle import clib
from oracle.refine_fp64 import refine_template_fp64, residuals_fp64
from paper_2203_10879_b200 import RefineConfig, RefineStatus, TriEqProblem, ZPlanar, inputs, ozaki, refine_template
from paper_2203_10879_b200 import solve_block

pytestmark = pytest.mark.gpu
U = 2.0 ** -53


def dd_exact(a, b):
    z = np.zeros(a.shape)
    pa = (np.ascontiguousarray(a.real), z, np.ascontiguousarray(a.imag), z.copy())
    z = np.zeros(b.shape)
    pb = (np.ascontiguousarray(b.real), z, np.ascontiguousarray(np.imag(b)), z.copy())
    o = clib.gemm_dd(pa, pb)
    return (o[0] + o[1]) + 1j * (o[2] + o[3])


def gauss_product(x, y):
    M, K = x.shape
    N = y.shape[1]
    pl = ozaki.gauss_plan(K, ozaki.HP_BETA, ozaki.HP_BETA)
    ea = ozaki.encode(ZPlanar.from_any(x), M, K, "a", pl)
    eb = ozaki.encode(ZPlanar.from_any(y), K, N, "b", pl)
    res = ozaki.ResidueBuffer(M, N, pl.nmod, "cuda")
    ozaki.gemm_residues(ea, eb, pl, res)
    out = ZPlanar.empty(M, N)
    ozaki.decode(res, ea, eb, pl, out)
    return out.to_numpy()


@pytest.mark.parametrize("M,N,K", [(96, 80, 130), (256, 200, 300)])
def test_graded_rows_and_columns_componentwise(M, N, K):
    rng = np.random.default_rng(M + N + K)
    d1 = np.exp2(rng.integers(-20, 21, M).astype(float))
    d2 = np.exp2(rng.integers(-20, 21, N).astype(float))
    a = (rng.standard_normal((M, K)) + 1j * rng.standard_normal((M, K))) * d1[:, None]
    b = (rng.standard_normal((K, N)) + 1j * rng.standard_normal((K, N))) * d2[None, :]
    exact = dd_exact(a, b)
    got = gauss_product(a, b)
    scale = np.abs(a) @ np.abs(b)
    # entry by entry, relative to the natural size of the entry: the grading
    # is absorbed by the per-row / per-column exponents
    assert np.max(np.abs(got - exact) / scale) <= 4 * U
    blas = a @ b
    assert np.max(np.abs(got - exact) / scale) <= max(2 * np.max(np.abs(blas - exact) / scale), 4 * U)


def test_graded_inside_rows_is_normwise():
    """Columns of A (the K direction) scaled by 2^+-20: inside one row the
    entries span 2^40, so the smallest lose bits — the error stays below the
    normwise bound 2^-beta sqrt(K) max|a_i.| max|b_.j| per entry (and the
    product's Frobenius error below BLAS's on the same inputs)."""
    rng = np.random.default_rng(9)
    M, N, K = 120, 90, 200
    dk = np.exp2(rng.integers(-20, 21, K).astype(float))
    a = (rng.standard_normal((M, K)) + 1j * rng.standard_normal((M, K))) * dk[None, :]
    b = rng.standard_normal((K, N)) + 1j * rng.standard_normal((K, N))
    exact = dd_exact(a, b)
    got = gauss_product(a, b)
    amax = np.abs(a).max(axis=1)
    bmax = np.abs(b).max(axis=0)
    bound = 2.0 ** -ozaki.HP_BETA * 4 * np.sqrt(K) * 2 * amax[:, None] * bmax[None, :]
    assert np.all(np.abs(got - exact) <= bound)
    assert np.linalg.norm(got - exact) <= max(2 * np.linalg.norm(a @ b - exact), 4 * U * np.linalg.norm(exact))


@pytest.mark.parametrize("n,seed", [(160, 7), (400, 8)])
def test_restore_full_sigma_matches_oracle(n, seed):
    a = inputs.gaussian_complex(n, seed)
    q = inputs.schur_vectors(a).astype(np.complex128)
    cfg = RefineConfig(precision="fp64", tol_factor=10.0 / n, max_iters=10, restore_full_sigma=True,
                       skip_final_ortho=False)
    pair, rep = refine_template(a, q, cfg)
    ref = refine_template_fp64(a, q, tol_factor=10.0 / n, max_iters=10, restore_full_sigma=True,
                               skip_final_ortho=False)
    assert rep.status.value == ref["status"] == "Converged"
    assert abs(rep.iterations - ref["iterations"]) <= 1
    assert rep.hp_matmul_count == 2 + 4 * rep.iterations and not rep.skip_fired
    rel_e, ortho = residuals_fp64(a, pair.q.cpu().numpy())
    assert rel_e <= 15 * U
    assert ortho <= 2 * max(residuals_fp64(a, ref["q"])[1], 10 * np.sqrt(n) * U)
    # and it agrees with the default two-product update to FP64 accuracy
    p2, r2 = refine_template(a, q, RefineConfig(precision="fp64", tol_factor=10.0 / n, max_iters=10,
                                                skip_final_ortho=False))
    assert r2.iterations == rep.iterations
    assert np.linalg.norm(p2.q.cpu().numpy() - pair.q.cpu().numpy()) <= 1e3 * U * np.sqrt(n)


def test_restore_full_sigma_dd_mode_converges():
    """dd mode with the two extra terms (the reference's own branch)."""
    from paper_2203_10879_b200 import verify_pair
    n = 96
    a = inputs.config4_matrix(n, 0, strict_scale=1.0 / np.sqrt(n))
    q = inputs.schur_vectors(a, np.complex128)
    pair, rep = refine_template(a, q, RefineConfig(precision="dd", max_iters=10, restore_full_sigma=True))
    assert rep.status is RefineStatus.CONVERGED
    v = verify_pair(a, pair)
    assert v.ortho_residual <= 1e-28 and v.tri_residual <= 10 * n * 2.0 ** -106 * np.linalg.norm(a)


def test_clip_counts_complex64_tensor_core_far_path_n2048():
    """Planted right-hand sides far above the clip threshold among a bulk far
    below it: the complex64 solve (far updates on tcgen05 kind::f16) clips
    exactly the entries the C restatement clips, at n = 2048."""
    n = 2048
    rng = np.random.default_rng(2048)
    t = np.triu(rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)))
    t[np.diag_indices(n)] = np.arange(n) * 1.1 + 1j * rng.standard_normal(n)
    e = np.tril(rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)), -1) * 1e-4
    planted = [(n - 1, 0), (n // 2, n // 3), (n - 40, n - 90), (1500, 700), (1999, 3), (900, 899)]
    for (i, j) in planted:
        e[i, j] = 1e6  # |l| >= 1e6 / |t_ii - t_jj| >> the threshold: clipped, so nothing cascades
    thr = 0.5
    t64, e64 = t.astype(np.complex64), e.astype(np.complex64)
    l_or, clipped_or = clib.solve_block(t64, e64, clip_threshold=thr, dtype=np.complex64)
    sol = solve_block(TriEqProblem(t=t64, e=e64, clip_threshold=thr), lp_dtype=torch.complex64)
    assert clipped_or == len(planted)
    assert sol.clipped_count == clipped_or, (sol.clipped_count, clipped_or)
    # the same entries are zero (the clipped ones) and the rest agree to complex64 level
    assert np.array_equal(sol.l == 0, l_or == 0)
    assert np.linalg.norm(sol.l - l_or) <= 1e-4 * np.linalg.norm(l_or)


def test_solve_n8192_matches_blas_port():
    """The complex64 solve at the bench size (n = 8192, tensor-core far
    updates with scaled two-piece FP16 operands, ~22 significant bits) against
    the BLAS-backed port of the reference solver (oracle/trisolve_blas.py,
    pinned to the C restatement) in complex64 and complex128 arithmetic: the
    GPU's error against the complex128 solution stays within 4x of the
    complex64 CPU port's own."""
    from oracle import trisolve_blas
    n = 8192
    rng = np.random.default_rng(8192)
    t = np.triu(rng.standard_normal((n, n)).astype(np.float32) + 1j * rng.standard_normal((n, n)).astype(np.float32))
    t[np.diag_indices(n)] = (np.arange(n) * 1.1 + 1j * rng.standard_normal(n)).astype(np.complex64)
    e = (np.tril(rng.standard_normal((n, n)).astype(np.float32), -1) * 1e-4).astype(np.complex64)
    t64 = t.astype(np.complex64)
    l_or = trisolve_blas.solve_block(t64, e, dtype=np.complex64)
    l_ref = trisolve_blas.solve_block(t64.astype(np.complex128), e.astype(np.complex128), dtype=np.complex128)
    sol = solve_block(TriEqProblem(t=t64, e=e), lp_dtype=torch.complex64)
    scale = np.linalg.norm(l_ref)
    err_gpu = np.linalg.norm(sol.l - l_ref) / scale
    err_port = np.linalg.norm(l_or - l_ref) / scale
    assert err_gpu <= 8 * err_port and err_gpu <= 1e-5, (err_gpu, err_port)
