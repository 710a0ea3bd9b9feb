"""The reference's public surface beyond refine_template, on the GPU
(reference __init__.py:1-102):

  * DDMatrix arithmetic, stril_extract and frobenius_norm — BIT-IDENTICAL to
    the reference (tests/golden/ddops_ref.*, made by the unmodified reference);
  * newton_schulz_step / merged_update — the reference's own contract tests
    restated (test_acceptance.py:214-252): the NS residual identity
    -3/4 D^2 + 1/4 D^3 to 1e-28, ortho <= 10 eps^4, move <= 10 eps^2;
  * solve_scalar / solve_block / stats (test_trisolve.py:380-398,
    test_acceptance.py:172-195): dense-operator oracle, separation errors,
    the invocation counters;
  * DDMatrix in, DDMatrix out: refine_template / verify_pair / matmul_hp take
    the reference's container (anything with .cells(), column-major) and
    results convert back with .to_ddmatrix().
"""
import numpy as np
import pytest
import torch

from paper_2203_10879_b200 import (
    DDMatrix,
    NormTooLarge,
    RefineConfig,
    RefineStatus,
    SeparationError,
    TriEqProblem,
    counters,
    frobenius_norm,
    matmul_hp,
    merged_update,
    newton_schulz_step,
    refine_template,
    reset_counters,
    reset_stats,
    solve_block,
    solve_scalar,
    stats,
    stril_extract,
    verify_pair,
)
from paper_2203_10879_b200.matrix import DDPlanar

pytestmark = pytest.mark.gpu
U_HP = 2.0 ** -106


def ddm(arr, name, k):
    return DDMatrix(*(arr["%s%s_%d" % (name, c, k)] for c in ("rh", "rl", "ih", "il")))


def test_dd_ops_bit_identical_to_reference(golden):
    meta, arr = golden("ddops_ref")
    for c in meta["cases"]:
        k = c["k"]
        a, b = ddm(arr, "a", k), ddm(arr, "b", k)
        assert (a + b).bits_equal(ddm(arr, "add", k)), c
        assert (a - b).bits_equal(ddm(arr, "sub", k)), c
        assert a.scale(c["s"]).bits_equal(ddm(arr, "scale", k)), c
        nrm = frobenius_norm(a)
        assert (nrm.hi, nrm.lo) == (c["norm_hi"], c["norm_lo"]), (c, nrm)
        # the device container gives the same bits
        nrm_d = frobenius_norm(a.to_device())
        assert (nrm_d.hi, nrm_d.lo) == (c["norm_hi"], c["norm_lo"])
        if c["m"] == c["n"]:
            e, t = stril_extract(a)
            assert e.bits_equal(ddm(arr, "stril_e", k)) and t.bits_equal(ddm(arr, "stril_t", k))
            assert (e + t).bits_equal(a)


def test_stril_extract_and_norm_lp_inputs():
    rng = np.random.default_rng(1)
    m = rng.standard_normal((9, 9)) + 1j * rng.standard_normal((9, 9))
    e, t = stril_extract(m)
    assert np.array_equal(e, np.tril(m, -1)) and np.array_equal(t, np.triu(m)) and e.flags.f_contiguous
    et, tt = stril_extract(torch.from_numpy(m).cuda())
    assert et.is_cuda and np.array_equal(et.cpu().numpy(), e)
    with pytest.raises(ValueError):
        stril_extract(np.ones((2, 3)))
    # lp matrix: the dd norm of its exact embedding
    assert float(frobenius_norm(m)) == float(frobenius_norm(DDMatrix.from_lp(m)))
    assert abs(float(frobenius_norm(m)) - np.linalg.norm(m)) <= 1e-15 * np.linalg.norm(m)


def dd_unitary(rng, n):
    """A dd-accurate random unitary: binary64 QR, then two dd Newton-Schulz
    steps (the reference builds it with qr_retract, test_refine.py:38-40)."""
    q0, _ = np.linalg.qr(rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)))
    return newton_schulz_step(newton_schulz_step(DDMatrix.from_lp(q0)))


def test_newton_schulz_residual_identity():
    """test_acceptance.py:239-252: one plain step on Q with Gram defect D
    leaves exactly -(3/4) D^2 + (1/4) D^3, up to pair rounding."""
    rng = np.random.default_rng(707)
    n = 12
    eye = DDMatrix.eye(n)
    for _ in range(5):
        q0, _ = np.linalg.qr(rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)))
        g = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
        h = (g + g.conj().T) / 2.0
        qp = DDMatrix.from_lp(q0 @ (np.eye(n) + 1e-3 * h))
        delta = matmul_hp(qp, qp, trans_a=True) - eye
        reset_counters()
        q_new = newton_schulz_step(qp)
        assert counters()["hp_calls"] == 2 and isinstance(q_new, DDMatrix)
        lhs = matmul_hp(q_new, q_new, trans_a=True) - eye
        d2 = matmul_hp(delta, delta)
        rhs = d2.scale(-0.75) + matmul_hp(d2, delta).scale(0.25)
        assert float(frobenius_norm(lhs - rhs)) <= 1e-28
    with pytest.raises(NormTooLarge):
        newton_schulz_step(DDMatrix.eye(4, 2.0))


@pytest.mark.parametrize("eps", [1e-3, 1e-5])
def test_merged_update_contract(eps):
    """test_acceptance.py:214-238 (NS strategy): ortho <= 10 eps^4 and the
    step moves Q(I + W) by <= 10 eps^2."""
    rng = np.random.default_rng(707)
    n = 12
    eye = DDMatrix.eye(n)
    for _ in range(10):
        q0, _ = np.linalg.qr(rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)))
        q = DDMatrix.from_lp(q0)
        g = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
        w = g - g.conj().T
        w *= eps / np.linalg.norm(w, "fro")
        target = matmul_hp(q, eye + DDMatrix.from_lp(w))
        y = matmul_hp(q, q, trans_a=True) - eye
        reset_counters()
        q_new = merged_update(q, w, y)
        assert counters()["hp_calls"] == 1
        ortho = float(frobenius_norm(matmul_hp(q_new, q_new, trans_a=True) - eye))
        move = float(frobenius_norm(q_new - target))
        assert ortho <= 10.0 * eps ** 4, ortho
        assert move <= 10.0 * eps ** 2, move
        # restore_full_sigma keeps W^2 Y + W^2 Y W: the same contract
        q_full = merged_update(q, w, y, restore_full_sigma=True)
        assert float(frobenius_norm(matmul_hp(q_full, q_full, trans_a=True) - eye)) <= 10.0 * eps ** 4


def test_merged_update_fp64_mode_matches_numpy():
    """FP64 operands: the FP64-mode update (complex64 lp products) against the
    restatement's merged_update (oracle/refine_fp64.py:70-89)."""
    from oracle.refine_fp64 import merged_update as oracle_update
    rng = np.random.default_rng(5)
    n = 64
    q, _ = np.linalg.qr(rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)))
    g = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    w = 1e-4 * (g - g.conj().T) / np.linalg.norm(g)
    y = q.conj().T @ q - np.eye(n)
    for full in (False, True):
        got = merged_update(q, w, y, restore_full_sigma=full).cpu().numpy()
        ref = oracle_update(q, w, y, full)
        assert np.linalg.norm(got - ref) <= 1e-13 * np.sqrt(n), np.linalg.norm(got - ref)
    # a general (not skew-Hermitian) W takes the full-product path
    w2 = 1e-4 * g / np.linalg.norm(g)
    got = merged_update(q, w2, y).cpu().numpy()
    assert np.linalg.norm(got - oracle_update(q, w2, y)) <= 1e-13 * np.sqrt(n)


def dense_commutator_solve(t, e):
    n = t.shape[0]
    pairs = [(i, j) for j in range(n - 1) for i in range(j + 1, n)]
    op = np.zeros((len(pairs), len(pairs)), dtype=complex)
    for col, (p, q) in enumerate(pairs):
        basis = np.zeros((n, n), dtype=complex)
        basis[p, q] = 1.0
        image = t @ basis - basis @ t
        for row, (i, j) in enumerate(pairs):
            op[row, col] = image[i, j]
    sol = np.linalg.solve(op, np.array([-e[i, j] for (i, j) in pairs]))
    l = np.zeros((n, n), dtype=complex)
    for v, (i, j) in zip(sol, pairs):
        l[i, j] = v
    return l


def test_solvers_match_dense_oracle_and_counters():
    """test_acceptance.py:172-195 (fewer draws) and test_trisolve.py:380-398."""
    rng = np.random.default_rng(505)
    for _ in range(20):
        n = int(rng.integers(3, 25))
        diag = np.cumsum(0.1 + rng.uniform(0.0, 0.4, size=n)) + 1j * rng.uniform(-5.0, 5.0, size=n)
        t = np.triu(rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)), 1) + np.diag(diag)
        e = np.tril(rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)), -1)
        scalar = solve_scalar(TriEqProblem(t=t, e=e))
        assert isinstance(scalar.l, np.ndarray) and scalar.l.dtype == np.complex128
        assert np.max(np.abs(scalar.l - dense_commutator_solve(t, e))) <= 1e-10
        block = solve_block(TriEqProblem(t=t, e=e), n_min=4)
        assert np.max(np.abs(block.l - scalar.l)) <= 1e-10
        dup = t.copy()
        i, j = sorted(rng.choice(n, size=2, replace=False))
        dup[j, j] = dup[i, i]
        with pytest.raises(SeparationError):
            solve_scalar(TriEqProblem(t=dup, e=e))
        with pytest.raises(SeparationError):
            solve_block(TriEqProblem(t=dup, e=e))
    t = np.triu(rng.standard_normal((16, 16)) + 0j, 1) + np.diag(np.arange(16) * 0.5 + 1.0)
    e = np.tril(rng.standard_normal((16, 16)) + 0j, -1)
    reset_stats()
    solve_scalar(TriEqProblem(t=t, e=e))
    assert stats() == {"scalar_solves": 1, "block_solves": 0, "sylvester_solves": 0}
    reset_stats()
    solve_block(TriEqProblem(t=t, e=e), n_min=4)
    assert stats() == {"scalar_solves": 0, "block_solves": 1, "sylvester_solves": 3}
    reset_stats()


def make_instance(rng, n):
    """test_refine.py:43-58: A = U T U^H with separated eigenvalues."""
    t = np.triu(0.5 * (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))), 1)
    t = t + np.diag(np.arange(n) + 0.7 * rng.random(n) + 1j * rng.uniform(-1.0, 1.0, n))
    u = dd_unitary(rng, n)
    a = matmul_hp(matmul_hp(u, DDMatrix.from_lp(t)), u, trans_b=True)
    return a, u


def perturbed_candidate(rng, u, eps):
    """test_refine.py:61-68."""
    n = u.rows
    x = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    k = x - x.conj().T
    k *= eps / np.linalg.norm(k, "fro")
    poly = np.eye(n) + k + k @ k / 2.0 + k @ k @ k / 6.0
    return matmul_hp(u, DDMatrix.from_lp(poly))


def dd_cfg(**kw):
    return RefineConfig(precision="dd", **kw)


def test_ddmatrix_in_ddmatrix_out_and_reference_cases():
    """Reference containers through the whole boundary, with the hot-path
    cases of test_refine.py restated: exact candidate (75-87), quadratic
    residual sequence (90-106), contraction near the fixed point (148-162)."""
    import math
    rng = np.random.default_rng(11)
    a, u = make_instance(rng, 4)
    pair, rep = refine_template(a, u, dd_cfg())
    assert rep.status is RefineStatus.CONVERGED and rep.iterations <= 1
    assert len(rep.residual_history) == rep.iterations + 1
    assert rep.residual_history[-1][0] <= 10.0 * 4 * U_HP * float(frobenius_norm(a))
    t = pair.t.to_ddmatrix()
    assert isinstance(t, DDMatrix) and t.re_hi.flags.f_contiguous
    e, _ = stril_extract(t)
    assert float(frobenius_norm(e)) == 0.0 and rep.wall_time > 0.0
    # quadratic residual sequence
    rng = np.random.default_rng(5)
    a, u = make_instance(rng, 8)
    qhat = perturbed_candidate(rng, u, 1e-4)
    pair, rep = refine_template(a, qhat, dd_cfg())
    assert rep.status is RefineStatus.CONVERGED
    norm_a = float(frobenius_norm(a))
    rel = [x / norm_a for x, _ in rep.residual_history]
    floor = 100.0 * 8 * U_HP
    exps = [math.log(r1) / math.log(r0) for r0, r1 in zip(rel[1:], rel[2:]) if r1 >= floor and r0 <= 1e-2]
    assert len(exps) >= 1 and all(x >= 1.8 for x in exps), rel
    # verify_pair on reference containers (the result converted back)
    host_pair = type(pair)(q=pair.q.to_ddmatrix(), t=pair.t.to_ddmatrix(), ortho_residual=pair.ortho_residual)
    v = verify_pair(a, host_pair)
    assert v.ortho_residual <= 1e-28 and v.tri_residual <= 2.0 * 10.0 * 8 * U_HP * norm_a
    # contraction near the fixed point
    rng = np.random.default_rng(41)
    a, u = make_instance(rng, 32)
    qhat = perturbed_candidate(rng, u, 1e-3)
    pair, rep = refine_template(a, qhat, dd_cfg())
    assert rep.status is RefineStatus.CONVERGED
    norm_a = float(frobenius_norm(a))
    floor = 100.0 * 32 * U_HP * norm_a
    hist = [x for x, _ in rep.residual_history[1:]]
    checked = 0
    for e0, e1 in zip(hist, hist[1:]):
        if floor <= e0 <= 1e-8 * norm_a:
            assert e1 <= max(1e-6 * e0, floor)
            checked += 1
    assert checked >= 1


def test_reference_error_and_status_cases():
    """test_refine.py:165-191 (validation) and 266-287 (non-finite + hint,
    clipping keeps the run alive)."""
    rng = np.random.default_rng(0)
    a, u = make_instance(rng, 4)
    with pytest.raises(ValueError):
        refine_template(a, DDMatrix.eye(5), dd_cfg())
    with pytest.raises(ValueError):
        refine_template(np.full((3, 3), np.nan), np.eye(3), dd_cfg())
    for bad in (dict(tol_factor=0.0), dict(max_iters=0), dict(n_min=1), dict(clip_threshold=-1e-5),
                dict(ortho="ns")):
        with pytest.raises(ValueError):
            RefineConfig(**bad)
    t0 = np.triu(np.ones((3, 3)), 1) + np.diag([0.0, 1e-200, 2e-200])
    a = t0 + 1e-3 * np.tril(np.ones((3, 3)), -1)
    pair, rep = refine_template(a, np.eye(3), dd_cfg())
    assert rep.status is RefineStatus.NON_FINITE and rep.iterations == 1
    assert len(rep.residual_history) == 2
    assert "iteration 1" in rep.detail and "clip_threshold" in rep.detail
    pair, rep = refine_template(a, np.eye(3), dd_cfg(clip_threshold=1e-5))
    assert rep.status is RefineStatus.MAX_ITERS and rep.iterations == 20
    assert rep.clipped_total == 3 * 20 and "clip_threshold" not in rep.detail


def test_verify_pair_exact_cases():
    """test_refine.py:349-371."""
    from paper_2203_10879_b200 import SchurPair
    a = DDMatrix.from_lp(np.array([[5.0]]))
    v = verify_pair(a, SchurPair(q=DDMatrix.eye(1), t=a, ortho_residual=0.0))
    assert v.ortho_residual == 0.0 and v.tri_residual == 0.0 and v.similarity_residual == 0.0
    rng = np.random.default_rng(13)
    a = DDMatrix.from_lp(rng.standard_normal((4, 4)) + 1j * rng.standard_normal((4, 4)))
    v = verify_pair(a, SchurPair(q=DDMatrix.eye(4), t=a, ortho_residual=0.0))
    e, _ = stril_extract(a)
    assert v.tri_residual == float(frobenius_norm(e))
    assert v.ortho_residual == 0.0 and v.similarity_residual == 0.0


def test_quadratic_convergence_order_acceptance():
    """test_acceptance.py:114-142."""
    import math
    rng = np.random.default_rng(11)
    n = 16
    t0 = np.triu(0.1 * (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))), 1)
    t0 += np.diag(np.arange(1.0, n + 1.0) + 0.25j * (-1.0) ** np.arange(n))
    q0, _ = np.linalg.qr(rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)))
    q_dd = newton_schulz_step(DDMatrix.from_lp(q0))
    a_dd = matmul_hp(matmul_hp(q_dd, DDMatrix.from_lp(t0)), q_dd.conj_t())
    for eps in (1e-3, 1e-4, 1e-5):
        g = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
        s = g - g.conj().T
        s *= eps / np.linalg.norm(s, "fro")
        qhat = matmul_hp(q_dd, DDMatrix.eye(n) + DDMatrix.from_lp(s))
        reset_counters()
        pair, rep = refine_template(a_dd, qhat, dd_cfg(seed=0))
        assert rep.status is RefineStatus.CONVERGED
        assert rep.hp_matmul_count == 2 + 4 * rep.iterations - (1 if rep.skip_fired else 0)
        es = [h[0] for h in rep.residual_history[1:]]
        kept = []
        for value in es:
            if value <= 1e-28:
                break
            kept.append(value)
        assert len(kept) >= 3, es
        orders = [math.log(kept[k + 1]) / math.log(kept[k]) for k in range(len(kept) - 1)]
        assert min(orders) >= 1.8, orders


def test_device_containers_stay_on_device():
    rng = np.random.default_rng(3)
    q0, _ = np.linalg.qr(rng.standard_normal((16, 16)) + 1j * rng.standard_normal((16, 16)))
    qd = DDMatrix.from_lp(q0).to_device()
    out = newton_schulz_step(qd)
    assert isinstance(out, DDPlanar)
    g = matmul_hp(out, out, trans_a=True)
    assert isinstance(g, DDPlanar)
    back = g.to_ddmatrix()
    assert np.abs(back.re_hi - np.eye(16)).max() <= 1e-15
