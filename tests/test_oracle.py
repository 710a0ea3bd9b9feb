"""Pins for the CPU oracle (oracle/) against the REAL reference's outputs.

Fixtures in tests/golden/ were produced by tests/golden/make_golden.py from
the unmodified reference package.  Known-answer cases restate the
reference's own unit tests (file:line cited per test).
"""
import numpy as np
import pytest

from oracle import clib
from oracle.refine_fp64 import refine_template_fp64, residuals_fp64


def dense_operator_solve(t, e):
    """Independent oracle: assemble L -> stril(T L - L T) on the n(n-1)/2
    strictly lower unknowns and solve densely (test_trisolve.py:35-69)."""
    n = t.shape[0]
    pairs = [(i, j) for j in range(n - 1) for i in range(j + 1, n)]
    idx = {pq: k for k, pq in enumerate(pairs)}
    op = np.zeros((len(pairs), len(pairs)), dtype=complex)
    for (i, j), row in idx.items():
        for (p, q), col in idx.items():
            v = 0j
            if q == j:
                v += t[i, p]
            if p == i:
                v -= t[q, j]
            op[row, col] = v
    sol = np.linalg.solve(op, np.array([-e[i, j] for (i, j) in pairs]))
    l = np.zeros((n, n), dtype=complex)
    for k, (i, j) in enumerate(pairs):
        l[i, j] = sol[k]
    return l


def test_trisolve_c128_matches_reference_golden(golden):
    meta, arr = golden("trisolve_ref")
    for c in meta["cases"]:
        k = c["k"]
        t, e, l_ref = arr["t_%d" % k], arr["e_%d" % k], arr["l_%d" % k]
        l, clipped = clib.solve_block(t, e, n_min=c["n_min"], clip_threshold=c["clip"])
        assert clipped == c["clipped"], c
        scale = max(np.abs(l_ref).max(), 1e-300)
        assert np.abs(l - l_ref).max() <= 1e-13 * scale, c


def test_trisolve_c64_matches_reference_golden(golden):
    meta, arr = golden("trisolve_ref")
    for c in meta["cases"]:
        if c["clip"] is not None:
            continue  # entries at the clip threshold may flip at complex64 rounding
        k = c["k"]
        t, e, l_ref = arr["t_%d" % k], arr["e_%d" % k], arr["l_%d" % k]
        l, _ = clib.solve_block(t, e, n_min=c["n_min"], dtype=np.complex64)
        err = np.linalg.norm(l - l_ref) / max(np.linalg.norm(l_ref), 1e-300)
        assert err <= 1e-5, (c, err)


def test_trisolve_dense_operator_oracle():
    rng = np.random.default_rng(7)
    for n in (2, 3, 6, 9):
        t = np.triu(rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)))
        t[np.diag_indices(n)] = np.arange(n) * 1.3 + 1j * rng.standard_normal(n)
        e = np.tril(rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)), -1)
        l, _ = clib.solve_block(t, e, n_min=2)
        assert np.allclose(l, dense_operator_solve(t, e), rtol=1e-11, atol=1e-12)


def test_trisolve_known_answers():
    # 2x2 entry formula, test_trisolve.py:112-118
    t = np.array([[0.0, 0.0], [0.0, 1.0]], dtype=complex)
    e = np.array([[0.0, 0.0], [0.5, 0.0]], dtype=complex)
    l, _ = clib.solve_block(t, e)
    assert l[1, 0] == -0.5 and l[0, 0] == 0 and l[0, 1] == 0 and l[1, 1] == 0
    # zero rhs -> zero solution
    rng = np.random.default_rng(0)
    t = np.triu(rng.standard_normal((7, 7))) + np.diag(np.arange(7.0)) * 3
    l, c = clib.solve_block(t.astype(complex), np.zeros((7, 7), complex))
    assert not l.any() and c == 0
    # exact duplicate diagonal -> SeparationError (trisolve.py:104-113)
    t = np.diag([1.0, 2.0, 1.0]).astype(complex)
    with pytest.raises(clib.SeparationError):
        clib.solve_block(t, np.tril(np.ones((3, 3)), -1).astype(complex))
    # near-zero separation overflows to a huge finite value (test_trisolve.py:282-287)
    t = np.diag([0.0, 1e-200]).astype(complex)
    e = np.array([[0, 0], [1.0, 0]], dtype=complex)
    l, _ = clib.solve_block(t, e)
    assert l[1, 0] == -1e200
    # overflow -> NonFiniteError
    t = np.diag([0.0, 1e-300]).astype(complex)
    e = np.array([[0, 0], [1e300, 0]], dtype=complex)
    with pytest.raises(clib.NonFiniteError):
        clib.solve_block(t, e)
    # empty / n = 1
    l, c = clib.solve_block(np.zeros((0, 0), complex), np.zeros((0, 0), complex))
    assert l.shape == (0, 0)
    l, c = clib.solve_block(np.ones((1, 1), complex), np.zeros((1, 1), complex))
    assert l[0, 0] == 0


def test_ddgemm_bit_identical_to_reference(golden):
    meta, arr = golden("ddgemm_ref")
    for c in meta["cases"]:
        k = c["k"]
        a = tuple(arr["a%s_%d" % (x, k)] for x in ("rh", "rl", "ih", "il"))
        b = tuple(arr["b%s_%d" % (x, k)] for x in ("rh", "rl", "ih", "il"))
        out = clib.gemm_dd(a, b)
        for x, o in zip(("rh", "rl", "ih", "il"), out):
            assert np.array_equal(o, arr["c%s_%d" % (x, k)]), (c, x)


def test_ddgemm_exact_small():
    # [[1,2],[3,4]] @ [[5,6],[7,8]] = [[19,22],[43,50]] (test_ddmatrix.py:82-87)
    z = np.zeros((2, 2))
    a = (np.array([[1.0, 2], [3, 4]]), z, z, z)
    b = (np.array([[5.0, 6], [7, 8]]), z, z, z)
    out = clib.gemm_dd(a, b)
    assert np.array_equal(out[0], [[19, 22], [43, 50]])
    assert not out[1].any() and not out[2].any() and not out[3].any()


def test_fp64_oracle_config1_matches_reference_iterations(golden):
    """Option 2 (FP64 restatement) against option 1 (the reference in dd
    with the FP64 stop rule) on config 1: iterations ±1, same status."""
    from paper_2203_10879_b200 import inputs
    meta, arr = golden("configs_ref")
    ref = [c for c in meta["cases"] if c["tag"] == "config1_n256"][0]
    a = inputs.gaussian_complex(256, 0)
    q = arr["qhat_config1_n256"].astype(np.complex128)
    out = refine_template_fp64(a, q, tol_factor=10.0 / 256, max_iters=10)
    assert out["status"] == ref["status"] == "Converged"
    assert abs(out["iterations"] - ref["iterations"]) <= 1
    rel_e, ortho = residuals_fp64(a, out["q"])
    u = 2.0 ** -53
    assert out["residual_history"][-1][0] / out["norm_a"] <= 10 * u
    assert ortho <= 40 * np.sqrt(256) * u
    # entry residual (row 1) agrees with the reference's dd measurement
    assert np.isclose(out["residual_history"][1][0], ref["residual_history"][1][0], rtol=1e-6)


@pytest.mark.parametrize("n,dtype", [(150, np.complex128), (300, np.complex64), (333, np.complex128)])
def test_blas_solver_port_matches_c_restatement(n, dtype):
    """oracle/trisolve_blas.py (the timed CPU baseline's solver: the same
    recursive halving on BLAS / LAPACK ?trsyl kernels) against the C
    restatement of trisolve.py: the same L up to rounding, and both satisfy
    the equation to working precision."""
    from oracle import trisolve_blas
    rng = np.random.Generator(np.random.Philox(77 + n))
    t = np.triu(rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)))
    t[np.diag_indices(n)] = np.arange(n) * (1.0 + 0.5j) + rng.uniform(0.0, 0.5, n)
    e = 1e-3 * np.tril(rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)), -1)
    t, e = t.astype(dtype), e.astype(dtype)
    l_c, _ = clib.solve_block(t, e, dtype=dtype)
    l_b = trisolve_blas.solve_block(t, e, dtype=dtype)
    u = np.finfo(np.float32 if dtype == np.complex64 else np.float64).eps
    assert np.linalg.norm(l_b - l_c) <= 100 * u * np.sqrt(n) * np.linalg.norm(l_c)
    tt = t.astype(np.complex128)
    for l in (l_b, l_c):
        r = np.tril(tt @ l - l @ tt, -1) + e
        assert np.linalg.norm(r) <= 100 * u * np.sqrt(n) * np.linalg.norm(e)
    with pytest.raises(clib.SeparationError):
        t2 = t.copy()
        t2[5, 5] = t2[7, 7]
        trisolve_blas.solve_block(t2, e, dtype=dtype)


def test_fp64_oracle_blas_solver_same_history():
    """refine_template_fp64(solver="blas") — the bench's CPU arm — follows the
    C-solver restatement's history (iterations equal, residuals to 1e-3)."""
    from paper_2203_10879_b200 import inputs
    n = 200
    a = inputs.gaussian_complex(n, 21)
    q = inputs.schur_vectors(a).astype(np.complex128)
    r_c = refine_template_fp64(a, q, tol_factor=10.0 / n, max_iters=10)
    r_b = refine_template_fp64(a, q, tol_factor=10.0 / n, max_iters=10, solver="blas")
    assert r_c["status"] == r_b["status"] == "Converged"
    assert r_c["iterations"] == r_b["iterations"]
    for (e1, y1), (e2, y2) in zip(r_c["residual_history"][:-1], r_b["residual_history"][:-1]):
        assert abs(e1 - e2) <= 1e-3 * e1 and abs(y1 - y2) <= 1e-3 * y1 + 1e-15
