"""GPU parity of the individual libsr kernels against numpy / the oracle.

Tolerances: FP64 products 1e-13 normwise (k * u64 growth at these sizes),
complex64 products 2e-6 normwise, complex64 solves 2e-5 against the
complex128 reference (golden fixtures), complex128 solves 1e-12.
"""
import numpy as np
import pytest
import torch

from oracle import clib
from paper_2203_10879_b200 import TriEqProblem, ZPlanar, matmul_hp, matmul_lp, solve_block
from paper_2203_10879_b200 import SeparationError, NonFiniteError
from paper_2203_10879_b200 import _lib
from paper_2203_10879_b200.matrix import lp_empty

pytestmark = pytest.mark.gpu


def rnd(rng, m, n, real=False):
    x = rng.standard_normal((m, n))
    return x if real else x + 1j * rng.standard_normal((m, n))


@pytest.mark.parametrize("m,n,k", [(1, 1, 1), (5, 7, 3), (64, 64, 64), (129, 65, 17), (256, 256, 256),
                                   (300, 200, 513)])
@pytest.mark.parametrize("trans_a", [False, True])
@pytest.mark.parametrize("b_real", [False, True])
def test_zgemm_f64(m, n, k, trans_a, b_real):
    rng = np.random.default_rng(m * 1000 + n + k)
    a = rnd(rng, k, m) if trans_a else rnd(rng, m, k)
    b = rnd(rng, k, n, real=b_real)
    ref = (a.conj().T if trans_a else a) @ b
    ref = 0.5 * ref
    if m == n:
        ref = ref - np.eye(m) * 0.25
    out = matmul_hp(ZPlanar.from_any(a), ZPlanar.from_any(b), trans_a=trans_a, alpha=0.5,
                    diag_shift=(-0.25 if m == n else 0.0))
    got = out.to_numpy()
    err = np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-300)
    assert err <= 1e-13, err


@pytest.mark.parametrize("m,n,k", [(1, 1, 1), (7, 5, 3), (64, 64, 64), (130, 70, 33), (512, 256, 300)])
def test_cgemm_c64(m, n, k):
    rng = np.random.default_rng(m + 7 * n + k)
    a = rnd(rng, m, k).astype(np.complex64)
    b = rnd(rng, k, n).astype(np.complex64)
    ref = a.astype(np.complex128) @ b.astype(np.complex128)
    ad = lp_empty(m, k)
    bd = lp_empty(k, n)
    ad[:, :k] = torch.from_numpy(a)
    bd[:, :n] = torch.from_numpy(b)
    out = matmul_lp(ad, bd, m, n, k)
    got = out[:, :n].cpu().numpy()
    err = np.linalg.norm(got - ref) / np.linalg.norm(ref)
    assert err <= 2e-6, err


def test_trisolve_matches_reference_golden(golden):
    meta, arr = golden("trisolve_ref")
    for c in meta["cases"]:
        k = c["k"]
        t, e, l_ref = arr["t_%d" % k], arr["e_%d" % k], arr["l_%d" % k]
        sol = solve_block(TriEqProblem(t=t, e=e, clip_threshold=c["clip"]), lp_dtype=torch.complex128)
        l = sol.l  # numpy in, numpy out (like the reference)
        assert sol.clipped_count == c["clipped"], c
        err = np.abs(l - l_ref).max() / max(np.abs(l_ref).max(), 1e-300)
        assert err <= 1e-12, (c, err)
        if c["clip"] is None:
            sol = solve_block(TriEqProblem(t=t, e=e), lp_dtype=torch.complex64)
            l = sol.l
            err = np.linalg.norm(l - l_ref) / max(np.linalg.norm(l_ref), 1e-300)
            assert err <= 2e-5, (c, err)
            # the default follows the operands (complex128, the reference's binary64 lp)
            assert solve_block(TriEqProblem(t=t, e=e)).l.dtype == np.complex128


@pytest.mark.parametrize("n", [33, 100, 257, 700, 1157])
def test_trisolve_c64_matches_oracle(n):
    rng = np.random.default_rng(n)
    t = np.triu(rnd(rng, n, n))
    t[np.diag_indices(n)] = np.arange(n) * 1.1 + 1j * rng.standard_normal(n)
    e = np.tril(rnd(rng, n, n), -1) * 1e-3
    l_or, _ = clib.solve_block(t, e, dtype=np.complex64)
    l_ref, _ = clib.solve_block(t, e, dtype=np.complex128)
    sol = solve_block(TriEqProblem(t=t, e=e), lp_dtype=torch.complex64)
    l = sol.l
    err = np.linalg.norm(l - l_ref) / np.linalg.norm(l_ref)
    err_or = np.linalg.norm(l_or - l_ref) / np.linalg.norm(l_ref)
    assert err <= max(10 * err_or, 1e-5), (err, err_or)
    # residual of the equation itself
    res = np.linalg.norm(np.tril(t @ l - l @ t, -1) + e) / np.linalg.norm(e)
    assert res <= 1e-4, res


@pytest.mark.parametrize("n", [291, 610])
def test_trisolve_c128_far_batches_match_oracle(n):
    """Sizes with several far batches (N >= 9 tiles): complex128 solve vs the
    C oracle to 1e-11, and the clip decisions (threshold between the bulk of
    |L| and a few planted large entries) identical."""
    rng = np.random.default_rng(n + 1)
    t = np.triu(rnd(rng, n, n))
    t[np.diag_indices(n)] = np.arange(n) * 1.1 + 1j * rng.standard_normal(n)
    e = np.tril(rnd(rng, n, n), -1) * 1e-3
    l_or, _ = clib.solve_block(t, e, dtype=np.complex128)
    sol = solve_block(TriEqProblem(t=t, e=e), lp_dtype=torch.complex128)
    l = sol.l
    err = np.linalg.norm(l - l_or) / np.linalg.norm(l_or)
    assert err <= 1e-11, err
    # clipping: plant a few large right-hand sides so their entries exceed the threshold
    e2 = e.copy()
    idx = [(n - 1, 0), (n // 2, n // 3), (n - 40, n - 90)]
    for (i, j) in idx:
        e2[i, j] = 1e3
    thr = 0.5
    l_or2, clipped_or = clib.solve_block(t, e2, clip_threshold=thr, dtype=np.complex128)
    sol2 = solve_block(TriEqProblem(t=t, e=e2, clip_threshold=thr), lp_dtype=torch.complex128)
    assert sol2.clipped_count == clipped_or and clipped_or >= 1
    l2 = sol2.l
    assert np.linalg.norm(l2 - l_or2) <= 1e-11 * np.linalg.norm(l_or2)


def test_trisolve_errors():
    t = np.diag([1.0, 2.0, 1.0]).astype(complex)
    with pytest.raises(SeparationError):
        solve_block(TriEqProblem(t=t, e=np.tril(np.ones((3, 3)), -1).astype(complex)))
    t = np.diag([0.0, 1e-300]).astype(complex)
    e = np.array([[0, 0], [1e300, 0]], dtype=complex)
    with pytest.raises(NonFiniteError):
        solve_block(TriEqProblem(t=t, e=e), lp_dtype=torch.complex128)
    # known answer (test_trisolve.py:112-118)
    t = np.array([[0.0, 0.0], [0.0, 1.0]], dtype=complex)
    e = np.array([[0.0, 0.0], [0.5, 0.0]], dtype=complex)
    l = solve_block(TriEqProblem(t=t, e=e), lp_dtype=torch.complex128).l
    assert l[1, 0] == -0.5 and l[0, 1] == 0


def test_split_norms_and_skew():
    rng = np.random.default_rng(3)
    n = 301
    m = rnd(rng, n, n)
    z = ZPlanar.from_any(m)
    t_lp = lp_empty(n)
    e_lp = lp_empty(n)
    scal = torch.zeros(4, dtype=torch.float64, device="cuda")
    red = torch.zeros(_lib.load().sr_reduce_workspace_bytes(), dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    _lib.call("sr_split_lp_c64", n, z.re_ptr(), z.im_ptr(), z.ld, t_lp.data_ptr(), e_lp.data_ptr(),
              t_lp.shape[1], scal.data_ptr(), red.data_ptr(), red.numel(), st)
    _lib.call("sr_fro_norm_f64", n, n, z.re_ptr(), z.im_ptr(), z.ld, scal.data_ptr() + 8, red.data_ptr(),
              red.numel(), st)
    s = scal.cpu().numpy()
    assert np.isclose(s[0], np.linalg.norm(np.tril(m, -1)), rtol=1e-14)
    assert np.isclose(s[1], np.linalg.norm(m), rtol=1e-14)
    assert np.array_equal(e_lp[:, :n].cpu().numpy(), np.tril(m, -1).astype(np.complex64))
    assert np.array_equal(t_lp[:, :n].cpu().numpy(), np.triu(m).astype(np.complex64))
    flags = torch.zeros(1, dtype=torch.int32, device="cuda")
    w = lp_empty(n)
    _lib.call("sr_skew_c64", n, e_lp.data_ptr(), e_lp.shape[1], w.data_ptr(), scal.data_ptr() + 16,
              flags.data_ptr(), red.data_ptr(), red.numel(), st)
    l = np.tril(m, -1).astype(np.complex64)
    wr = l - l.conj().T
    assert np.array_equal(w[:, :n].cpu().numpy(), wr)
    assert np.isclose(scal[2].item(), np.linalg.norm(wr.astype(np.complex128)), rtol=1e-12)
    assert flags.item() == 0
    # determinism: same launch twice, bitwise-equal norm
    _lib.call("sr_fro_norm_f64", n, n, z.re_ptr(), z.im_ptr(), z.ld, scal.data_ptr() + 24, red.data_ptr(),
              red.numel(), st)
    assert scal[3].item() == scal[1].item()


def test_sigma_merged_matches_numpy():
    rng = np.random.default_rng(5)
    n = 77
    w = (rnd(rng, n, n) * 1e-3).astype(np.complex64)
    y = rnd(rng, n, n) * 1e-6
    yw = (y.astype(np.complex64) @ w)
    w2 = w @ w
    w3 = w2 @ w
    ref = 2 * np.eye(n) + 2.0 * w.astype(np.complex128)
    ref = ref - y
    ref = ref - yw.astype(np.complex128)
    ref = ref + w2.astype(np.complex128)
    ref = ref + w3.astype(np.complex128)

    def dev(x):
        d = lp_empty(n)
        d[:, :n] = torch.from_numpy(x)
        return d
    wd, ywd, w2d, w3d = dev(w), dev(yw), dev(w2), dev(w3)
    yz = ZPlanar.from_any(y)
    s = ZPlanar.empty(n)
    _lib.call("sr_sigma_merged_f64", n, n, wd.data_ptr(), yz.re_ptr(), yz.im_ptr(), yz.ld, ywd.data_ptr(),
              w2d.data_ptr(), w3d.data_ptr(), None, None, wd.shape[1], s.re_ptr(), s.im_ptr(), s.ld,
              1, torch.cuda.current_stream().cuda_stream)
    assert np.array_equal(s.to_numpy(), ref)


def test_fused_update_forms_without_negligible_terms():
    """The fused update's kernels with the lp terms left out (products.lp_skips):
    X = Y - W (w2 = NULL) and S' = 2W - Y (yw = NULL), bit for bit; the full
    fused forms next to them; a dropped X W beside separate W^2, W^3 is rejected."""
    rng = np.random.default_rng(6)
    n = 61
    w = (rnd(rng, n, n) * 1e-5).astype(np.complex64)
    y = rnd(rng, n, n) * 1e-9
    w2 = (w @ w)
    st = torch.cuda.current_stream().cuda_stream

    def dev(x):
        d = lp_empty(n)
        d[:, :n] = torch.from_numpy(x)
        return d
    wd, w2d = dev(w), dev(w2)
    yz = ZPlanar.from_any(y)
    xd = lp_empty(n)
    _lib.call("sr_fused_lp_operand_c64", n, yz.re_ptr(), yz.im_ptr(), yz.ld, wd.data_ptr(), None, wd.shape[1],
              xd.data_ptr(), st)
    x_ref = (y - w.astype(np.complex128)).astype(np.complex64)
    assert np.array_equal(xd[:, :n].cpu().numpy(), x_ref)
    _lib.call("sr_fused_lp_operand_c64", n, yz.re_ptr(), yz.im_ptr(), yz.ld, wd.data_ptr(), w2d.data_ptr(),
              wd.shape[1], xd.data_ptr(), st)
    x_ref = ((y - w.astype(np.complex128)) - w2.astype(np.complex128)).astype(np.complex64)
    assert np.array_equal(xd[:, :n].cpu().numpy(), x_ref)
    s = ZPlanar.empty(n)
    _lib.call("sr_sigma_merged_f64", n, n, wd.data_ptr(), yz.re_ptr(), yz.im_ptr(), yz.ld, None, None, None, None,
              None, wd.shape[1], s.re_ptr(), s.im_ptr(), s.ld, 0, st)
    assert np.array_equal(s.to_numpy(), 2.0 * w.astype(np.complex128) - y)
    rc = _lib.load().sr_sigma_merged_f64(n, n, wd.data_ptr(), yz.re_ptr(), yz.im_ptr(), yz.ld, None, w2d.data_ptr(),
                                         w2d.data_ptr(), None, None, wd.shape[1], s.re_ptr(), s.im_ptr(), s.ld, 0, st)
    assert rc == _lib.SR_EINVAL
