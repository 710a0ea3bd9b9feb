"""GPU parity of refine_template (FP64 mode) against both oracles:
option 1 = the reference itself (dd, FP64 stop rule via tol_factor,
tests/golden/configs_ref.json) and option 2 = the FP64 restatement
(oracle/refine_fp64.py) run here on the same seeded inputs.

Tolerances: same status, iterations ±1, final relE below the
stop rule 10·u64, ||Q^H Q - I||_F within 2x of the restatement's value
(both measured by the same FP64 evaluator).
"""
import numpy as np
import pytest
import torch

from oracle.refine_fp64 import refine_template_fp64, residuals_fp64
from paper_2203_10879_b200 import NormTooLarge, RefineConfig, RefineStatus, SeparationError, inputs, refine_template

pytestmark = pytest.mark.gpu
U = 2.0 ** -53


def run_pair(a, q, n, **kw):
    cfg = RefineConfig(precision="fp64", tol_factor=10.0 / n, max_iters=10, **kw)
    pair, rep = refine_template(a, q, cfg)
    ref = refine_template_fp64(a, q, tol_factor=10.0 / n, max_iters=10, **kw)
    return pair, rep, ref


def check_parity(a, pair, rep, ref, n):
    assert rep.status.value == ref["status"], (rep.status, ref["status"])
    assert abs(rep.iterations - ref["iterations"]) <= 1
    assert len(rep.residual_history) == rep.iterations + 1
    q = pair.q.cpu().numpy()
    rel_e, ortho = residuals_fp64(a, q)
    rel_e_o, ortho_o = residuals_fp64(a, ref["q"])
    if rep.status is RefineStatus.CONVERGED:
        assert rep.residual_history[-1][0] / ref["norm_a"] <= 10 * U
        assert rel_e <= 10 * U * 1.5, rel_e
    assert ortho <= 2 * max(ortho_o, 10 * np.sqrt(n) * U), (ortho, ortho_o)
    # the hp-GEMM budget 2 + 4k (- 1 when the skip fires), refine.py:7-10
    assert rep.hp_matmul_count == 2 + 4 * rep.iterations - (1 if rep.skip_fired else 0)
    t = pair.t.cpu().numpy()
    assert not np.tril(t, -1).any()


def test_config1_matches_both_oracles(golden):
    meta, arr = golden("configs_ref")
    refc = [c for c in meta["cases"] if c["tag"] == "config1_n256"][0]
    n = 256
    a = inputs.gaussian_complex(n, 0)
    q = arr["qhat_config1_n256"].astype(np.complex128)
    pair, rep, ref = run_pair(a, q, n)
    check_parity(a, pair, rep, ref, n)
    assert rep.status.value == refc["status"]
    assert abs(rep.iterations - refc["iterations"]) <= 1
    # entry residual agrees with the reference's dd measurement of the same state
    assert np.isclose(rep.residual_history[1][0], refc["residual_history"][1][0], rtol=1e-6)


@pytest.mark.parametrize("n,seed", [(8, 1), (33, 2), (100, 3), (200, 4), (512, 5)])
def test_random_complex_matches_oracle(n, seed):
    a = inputs.gaussian_complex(n, seed)
    q = inputs.schur_vectors(a).astype(np.complex128)
    pair, rep, ref = run_pair(a, q, n)
    check_parity(a, pair, rep, ref, n)


@pytest.mark.parametrize("gemm", ["ozaki_std", "dmma"])
@pytest.mark.parametrize("n,seed", [(100, 3), (300, 6)])
def test_product_backends_match_oracle(gemm, n, seed):
    """The non-default product backends — (re, im)-plane Ozaki products and
    FP64 DMMA — against the FP64 restatement; the (re, im)-plane run meets the
    full parity bar and agrees with the Gaussian-CRT default to FP64 accuracy."""
    a = inputs.gaussian_complex(n, seed)
    q = inputs.schur_vectors(a).astype(np.complex128)
    cfg = RefineConfig(precision="fp64", tol_factor=10.0 / n, max_iters=10, gemm=gemm)
    pair, rep = refine_template(a, q, cfg)
    ref = refine_template_fp64(a, q, tol_factor=10.0 / n, max_iters=10)
    if gemm == "dmma":
        # FP64 DMMA accumulation noise on stril(Q^H A Q) grows like sqrt(n)
        # and can sit above the 10 u64 stop rule (the reason
        # the products are Ozaki-II), so the bar here is the noise floor
        rel_e, ortho = residuals_fp64(a, pair.q.cpu().numpy())
        assert rel_e <= 50 * 10 * U, rel_e
        assert ortho <= 10 * max(residuals_fp64(a, ref["q"])[1], 10 * np.sqrt(n) * U), ortho
        return
    check_parity(a, pair, rep, ref, n)
    pg, rg = refine_template(a, q, RefineConfig(precision="fp64", tol_factor=10.0 / n, max_iters=10))
    assert rg.iterations == rep.iterations
    assert np.linalg.norm(pg.q.cpu().numpy() - pair.q.cpu().numpy()) <= 1e3 * U * np.sqrt(n)


def test_real_a_config3_shape():
    n = 384
    a = inputs.gaussian_real(n, 0)
    q = inputs.schur_vectors(a).astype(np.complex128)
    pair, rep, ref = run_pair(a, q, n)
    check_parity(a, pair, rep, ref, n)


def test_clip_threshold_counts_like_oracle():
    n = 64
    a = inputs.gaussian_complex(n, 9)
    q = inputs.schur_vectors(a).astype(np.complex128)
    # a threshold above every correction entry: nothing clipped, normal run
    pair, rep, ref = run_pair(a, q, n, clip_threshold=1e-2)
    assert rep.status.value == ref["status"] == "Converged"
    assert rep.clipped_total == ref["clipped_total"] == 0
    # a threshold below every entry: everything clipped, no progress — both
    # runs end without converging (the exact failure status depends on the
    # rounding noise each precision pair sees once the correction is gone)
    pair, rep, ref = run_pair(a, q, n, clip_threshold=1e-14)
    assert rep.clipped_total > 0 and ref["clipped_total"] > 0
    assert rep.status.value in ("MaxIters", "Diverged") and ref["status"] in ("MaxIters", "Diverged")


def test_exact_candidate_and_errors():
    # A upper triangular, Q = I: converges at once (test_refine.py:75-90)
    rng = np.random.default_rng(0)
    n = 16
    t = np.triu(rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)))
    t[np.diag_indices(n)] = np.arange(n) + 1.0
    pair, rep = refine_template(t, np.eye(n), RefineConfig(precision="fp64"))
    # structural exit (refine.py:239-252): zero iterations, T built entrywise
    assert rep.status is RefineStatus.CONVERGED and rep.iterations == 0
    assert rep.hp_matmul_count == 2 and len(rep.residual_history) == 1
    assert np.array_equal(pair.t.cpu().numpy(), t)
    # a generic unitary candidate converges in at most one iteration
    rng2 = np.random.default_rng(1)
    u, _ = np.linalg.qr(rng2.standard_normal((n, n)) + 1j * rng2.standard_normal((n, n)))
    a = (u @ t) @ u.conj().T
    pair, rep = refine_template(a, u, RefineConfig(precision="fp64", tol_factor=10.0 / n))
    assert rep.status is RefineStatus.CONVERGED and rep.iterations <= 1
    # exactly repeated diagonal of T^ (Q = I, A not exactly triangular so the
    # structural exit does not apply): SeparationError propagates (refine.py:368-369)
    a2 = np.array([[1.0, 0.5, 0.0], [1e-3, 1.0, 0.0], [0.0, 0.0, 3.0]], dtype=complex)
    with pytest.raises(SeparationError):
        refine_template(a2, np.eye(3), RefineConfig(precision="fp64"))
    with pytest.raises(ValueError):
        refine_template(np.ones((3, 4)), np.eye(3), RefineConfig(precision="fp64"))
    with pytest.raises(ValueError):
        bad = np.eye(3)
        bad[0, 0] = np.nan
        refine_template(bad, np.eye(3), RefineConfig(precision="fp64"))
    with pytest.raises(ValueError):  # A is validated before the candidate's norm guard
        refine_template(bad, 4.0 * np.eye(3), RefineConfig(precision="fp64"))
    with pytest.raises(NormTooLarge):
        refine_template(np.eye(3), 4.0 * np.eye(3), RefineConfig(precision="fp64"))


def test_seed_determinism():
    n = 128
    a = inputs.gaussian_complex(n, 11)
    q = inputs.schur_vectors(a).astype(np.complex128)
    cfg = RefineConfig(precision="fp64", tol_factor=10.0 / n, max_iters=10)
    p1, r1 = refine_template(a, q, cfg)
    p2, r2 = refine_template(a, q, cfg)
    assert r1.residual_history == r2.residual_history
    assert torch.equal(p1.q, p2.q)


def test_config5_continuation_matches_oracle_chain():
    """Config 5 shape (smaller n): A(t_j) = A0 + t_j A1, each step started from
    the previous refined Q; the oracle runs the same chain on the CPU."""
    from paper_2203_10879_b200 import refine_continuation
    n, steps = 96, 5
    a0, a1 = inputs.config5_pair(n, 0)
    ts = [0.01 * j / 64 for j in range(steps)]
    q0 = inputs.schur_vectors(a0).astype(np.complex128)
    cfg = RefineConfig(precision="fp64", tol_factor=10.0 / n, max_iters=10)
    chain = refine_continuation(a0, a1, ts, q0, cfg)
    q = q0
    for (t, pair, rep), tj in zip(chain, ts):
        a = a0 + tj * a1
        ref = refine_template_fp64(a, q, tol_factor=10.0 / n, max_iters=10)
        q = ref["q"]
        assert rep.status.value == ref["status"] == "Converged"
        assert abs(rep.iterations - ref["iterations"]) <= 1
        rel_e, ortho = residuals_fp64(a, pair.q.cpu().numpy())
        assert rel_e <= 15 * U and ortho <= 2 * max(residuals_fp64(a, ref["q"])[1], 10 * np.sqrt(n) * U)


def test_host_result_matches_device_result():
    """refine_template(out=(q_host, t_host)): host Q, T identical to the
    device result (the speculative Q copy is the final Q)."""
    from paper_2203_10879_b200 import inputs
    n = 300
    a = inputs.gaussian_complex(n, 4)
    q = inputs.schur_vectors(a).astype(np.complex128)
    cfg = RefineConfig(precision="fp64", tol_factor=10.0 / n, max_iters=10)
    p1, r1 = refine_template(a, q, cfg)
    host = lambda: (torch.empty((n, n), dtype=torch.complex128, pin_memory=True),  # noqa: E731
                    torch.empty((n, n), dtype=torch.complex128, pin_memory=True))
    out = host()
    p2, r2 = refine_template(a, q, cfg, out=out)
    assert p2.q is out[0] and p2.t is out[1]
    assert torch.equal(p1.q.cpu(), p2.q) and torch.equal(p1.t.cpu(), p2.t)
    assert r1.iterations == r2.iterations and r1.residual_history == r2.residual_history
    # a run whose last step is an update (no skip): the final Q is the updated one
    cfg2 = RefineConfig(precision="fp64", tol_factor=10.0 / n, max_iters=10, skip_final_ortho=False)
    p3, _ = refine_template(a, q, cfg2)
    p4, _ = refine_template(a, q, cfg2, out=host())
    assert torch.equal(p3.q.cpu(), p4.q) and torch.equal(p3.t.cpu(), p4.t)


def test_host_inputs_match_device_inputs():
    """Host inputs land in the workspace's buffers (no per-call allocation):
    numpy, pinned torch and device-resident inputs give identical results,
    real A stays real, and a non-finite host Q^ still raises ValueError."""
    from paper_2203_10879_b200 import ZPlanar, inputs
    n = 256
    cfg = RefineConfig(precision="fp64", tol_factor=10.0 / n, max_iters=10)
    a = inputs.gaussian_real(n, 3)
    q = inputs.schur_vectors(a).astype(np.complex128)
    p_dev, r_dev = refine_template(ZPlanar.from_any(a), ZPlanar.from_any(q), cfg)
    q_dev, t_dev = p_dev.q.cpu(), p_dev.t.cpu()
    for aa, qq in ((a, q), (torch.from_numpy(a).pin_memory(), torch.from_numpy(q).pin_memory())):
        for _ in range(2):  # second call reuses the landing buffers
            p, r = refine_template(aa, qq, cfg)
            assert torch.equal(p.q.cpu(), q_dev) and torch.equal(p.t.cpu(), t_dev)
            assert r.residual_history == r_dev.residual_history
    bad = q.copy()
    bad[3, 7] = np.nan
    with pytest.raises(ValueError):
        refine_template(a, bad, cfg)
    bad_a = a.copy()
    bad_a[1, 1] = np.inf
    with pytest.raises(ValueError):
        refine_template(bad_a, q, cfg)


def test_host_inputs_fortran_order():
    """Fortran-ordered host inputs (LAPACK outputs) are transposed on the
    device, with results identical to C-ordered ones."""
    from paper_2203_10879_b200 import inputs
    n = 200
    cfg = RefineConfig(precision="fp64", tol_factor=10.0 / n, max_iters=10)
    for a in (inputs.gaussian_real(n, 5), inputs.gaussian_complex(n, 5)):
        q = inputs.schur_vectors(a).astype(np.complex128)
        p_c, r_c = refine_template(np.ascontiguousarray(a), np.ascontiguousarray(q), cfg)
        p_f, r_f = refine_template(np.asfortranarray(a), np.asfortranarray(q), cfg)
        p_t, r_t = refine_template(torch.from_numpy(np.asfortranarray(a)), torch.from_numpy(np.asfortranarray(q)), cfg)
        assert torch.equal(p_c.q.cpu(), p_f.q.cpu()) and torch.equal(p_c.t.cpu(), p_f.t.cpu())
        assert torch.equal(p_c.q.cpu(), p_t.q.cpu())
        assert r_c.residual_history == r_f.residual_history == r_t.residual_history


def test_negligible_lp_products_do_not_change_the_run(monkeypatch):
    """products.lp_skips leaves out lp products below their own error budget
    (the late updates' W^2 and X W); the run forming every product
    (SR_LP_SKIP=0) has the same status, iterations and residual history to
    measurement noise, and the same Q to a few units of roundoff."""
    n = 300
    a = inputs.gaussian_complex(n, 11)
    q = inputs.schur_vectors(a).astype(np.complex128)
    cfg = RefineConfig(precision="fp64", tol_factor=10.0 / n, max_iters=10)
    monkeypatch.setenv("SR_LP_SKIP", "0")
    pair0, rep0 = refine_template(a, q, cfg)
    monkeypatch.delenv("SR_LP_SKIP")
    pair1, rep1 = refine_template(a, q, cfg)
    assert rep1.status is rep0.status is RefineStatus.CONVERGED
    assert rep1.iterations == rep0.iterations
    na = np.linalg.norm(a)
    for (e0, y0), (e1, y1) in zip(rep0.residual_history, rep1.residual_history):
        assert abs(e0 - e1) <= 4 * U * na + 1e-6 * e0
        assert abs(y0 - y1) <= 40 * np.sqrt(n) * U + 1e-6 * y0
    dq = (pair0.q - pair1.q).abs().max().item()
    assert dq <= 16 * U, dq
