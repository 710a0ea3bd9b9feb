"""dd mode (the reference's own precision pair: hp = double-double, lp =
binary64) against the reference's golden runs (tests/golden/refine_dd_ref.*,
configs_ref.* — produced by the unmodified ddschur.refine_template) and the
oracle's bit-exact restatement of the reference dd GEMM.

Tolerances: dd products within 2^-96 normwise of the reference dd GEMM;
refinement: same status, iterations ±1, ||Q^H Q - I||_F <= 1e-28 and
||stril(Q^H A Q)||_F <= 10 n 2^-106 ||A||_F (test_acceptance.py:48-49)."""
import numpy as np
import pytest
import torch

from oracle import clib
from paper_2203_10879_b200 import RefineConfig, RefineStatus, ozaki, refine_template
from paper_2203_10879_b200.matrix import DDPlanar

pytestmark = pytest.mark.gpu
U_HP = 2.0 ** -106


def two_sum(a, b):
    s = a + b
    bb = s - a
    return s, (a - (s - bb)) + (b - bb)


def rand_dd(rng, shape):
    hi = rng.standard_normal(shape)
    lo = rng.standard_normal(shape) * 2.0 ** -55
    h, l = two_sum(hi, lo)
    hi2 = rng.standard_normal(shape)
    lo2 = rng.standard_normal(shape) * 2.0 ** -55
    h2, l2 = two_sum(hi2, lo2)
    return (h, l, h2, l2)  # re_hi, re_lo, im_hi, im_lo


def conj_t(p):
    return (p[0].T.copy(), p[1].T.copy(), -p[2].T, -p[3].T)


def dd_value(p):
    """complex value as (hi-sum) for error measurement: returns (big, small) parts."""
    return p[0] + 1j * p[2], p[1] + 1j * p[3]


def dd_diff_norm(a, b):
    ah, al = dd_value(a)
    bh, bl = dd_value(b)
    return np.linalg.norm((ah - bh) + (al - bl))


@pytest.mark.parametrize("m,n,k,trans", [(16, 16, 16, False), (64, 48, 40, True), (130, 70, 200, False)])
def test_dd_product_matches_reference_gemm(m, n, k, trans):
    rng = np.random.default_rng(m + n + k)
    a = rand_dd(rng, (k, m) if trans else (m, k))
    b = rand_dd(rng, (k, n))
    ref = clib.gemm_dd(conj_t(a) if trans else a, b)
    pl = ozaki.plan(k, ozaki.DD_BETA, ozaki.DD_BETA)
    ad, bd = DDPlanar.from_any(a), DDPlanar.from_any(b)
    ea = ozaki.encode(ad, ad.rows, ad.cols, "a", pl, conj_t=trans)
    eb = ozaki.encode(bd, bd.rows, bd.cols, "b", pl)
    res = ozaki.ResidueBuffer(m, n, pl.nmod, "cuda")
    ozaki.gemm_residues(ea, eb, pl, res)
    out = DDPlanar.empty(m, n)
    ozaki.decode(res, ea, eb, pl, out)
    got = out.to_numpy_cells()
    scale = np.linalg.norm(ref[0] + 1j * ref[2])
    assert dd_diff_norm(got, ref) <= 2.0 ** -96 * scale


def verify_dd(a_cells, q_cells):
    """verify_pair (refine.py:456-476) in dd on the CPU oracle: (ortho, tri)."""
    n = a_cells[0].shape[0]
    g = clib.gemm_dd(conj_t(q_cells), q_cells)
    gh, gl = dd_value(g)
    ortho = np.linalg.norm((gh - np.eye(n)) + gl)
    p = clib.gemm_dd(conj_t(q_cells), a_cells)
    t = clib.gemm_dd(p, q_cells)
    th, tl = dd_value(t)
    tri = np.linalg.norm(np.tril(th, -1) + np.tril(tl, -1))
    return ortho, tri


def cells(arr, name, k):
    return tuple(arr["%s%s_%d" % (name, c, k)] for c in ("rh", "rl", "ih", "il"))


def test_refine_dd_matches_reference_golden(golden):
    meta, arr = golden("refine_dd_ref")
    for c in meta["cases"]:
        k, n = c["k"], c["n"]
        a, qhat = cells(arr, "a", k), cells(arr, "qhat", k)
        pair, rep = refine_template(a, qhat, RefineConfig(precision="dd"))
        assert rep.status.value == c["status"], (c, rep.status)
        assert abs(rep.iterations - c["iterations"]) <= 1, (c, rep.iterations)
        assert len(rep.residual_history) == rep.iterations + 1
        assert rep.hp_matmul_count == 2 + 4 * rep.iterations - (1 if rep.skip_fired else 0)
        ortho, tri = verify_dd(a, pair.q.to_numpy_cells())
        norm_a = np.linalg.norm(a[0] + 1j * a[2])
        assert ortho <= 1e-28, (c, ortho)
        assert tri <= 10 * n * U_HP * norm_a, (c, tri)
        # history row 0 is the binary64 entry measurement, as in the reference
        assert np.isclose(rep.residual_history[0][0], c["residual_history"][0][0], rtol=0.1, atol=1e-30)


@pytest.mark.parametrize("m,n,k,trans", [(16, 16, 16, False), (64, 48, 40, True), (130, 70, 200, False)])
def test_dd_fma_product_matches_reference_gemm(m, n, k, trans):
    """The FMA-EFT dd GEMM (the measured alternative to the Ozaki dd
    products) against the bit-exact restatement of the reference dd GEMM."""
    from paper_2203_10879_b200.matmul import matmul_dd_fma
    rng = np.random.default_rng(m * n + k)
    a = rand_dd(rng, (k, m) if trans else (m, k))
    b = rand_dd(rng, (k, n))
    ref = clib.gemm_dd(conj_t(a) if trans else a, b)
    c = matmul_dd_fma(DDPlanar.from_any(a), DDPlanar.from_any(b), trans_a=trans)
    got = c.to_numpy_cells()
    scale = np.linalg.norm(ref[0] + 1j * ref[2])
    assert dd_diff_norm(got, ref) <= 2.0 ** -96 * scale, dd_diff_norm(got, ref) / scale


def test_refine_dd_config4_failure_mode_parity(golden):
    """BASELINE config 4 as written diverges in the reference:
    parity is on the status (±1 iteration); the well-conditioned variant
    converges."""
    from paper_2203_10879_b200 import inputs
    meta, arr = golden("configs_ref")
    for c in meta["cases"]:
        if not c["tag"].startswith("config4"):
            continue
        n = c["n"]
        scale = 1.0 / np.sqrt(n) if c["tag"].startswith("config4wc") else 1.0
        a = inputs.config4_matrix(n, 0, strict_scale=scale)
        q = arr["qhat_" + c["tag"]]
        pair, rep = refine_template(a, q, RefineConfig(precision="dd", max_iters=10))
        assert rep.status.value == c["status"], (c["tag"], rep.status, c["status"])
        assert abs(rep.iterations - c["iterations"]) <= 1, (c["tag"], rep.iterations, c["iterations"])
        if rep.status is RefineStatus.CONVERGED:
            ortho, tri = verify_dd((a.real.copy(), np.zeros((n, n)), a.imag.copy(), np.zeros((n, n))),
                                   pair.q.to_numpy_cells())
            assert ortho <= 1e-28 and tri <= 10 * n * U_HP * np.linalg.norm(a)


def test_verify_pair_dd_matches_cpu_dd_evaluator(golden):
    """verify_pair (refine.py:456-476) on the GPU in dd against the CPU dd
    evaluator built on the bit-exact reference dd GEMM: at the dd noise floor
    for refined pairs (the reference's acceptance bounds), and to 1e-8
    relative on a pair perturbed well above it."""
    from paper_2203_10879_b200 import SchurPair, verify_pair
    meta, arr = golden("refine_dd_ref")
    c = meta["cases"][0]
    k, n = c["k"], c["n"]
    a, qhat = cells(arr, "a", k), cells(arr, "qhat", k)
    pair, rep = refine_template(a, qhat, RefineConfig(precision="dd"))
    v = verify_pair(a, pair)
    norm_a = np.linalg.norm(a[0] + 1j * a[2])
    assert v.ortho_residual <= 1e-28 and v.tri_residual <= 10 * n * U_HP * norm_a
    assert v.similarity_residual <= 10 * n * U_HP * norm_a
    # perturb Q: residuals ~1e-20, far above both evaluators' floors
    rng = np.random.default_rng(3)
    qc = list(pair.q.to_numpy_cells())
    qc[1] = qc[1] + 1e-20 * rng.standard_normal(qc[1].shape)  # in the lo planes: below an ulp of hi
    qc[3] = qc[3] + 1e-20 * rng.standard_normal(qc[3].shape)
    qc = tuple(np.ascontiguousarray(x) for x in qc)
    v2 = verify_pair(a, SchurPair(q=qc, t=pair.t, ortho_residual=0.0))
    o_cpu, t_cpu = verify_dd(a, qc)
    assert abs(v2.ortho_residual - o_cpu) <= 1e-8 * o_cpu, (v2.ortho_residual, o_cpu)
    assert abs(v2.tri_residual - t_cpu) <= 1e-8 * t_cpu, (v2.tri_residual, t_cpu)
    # FP64 evaluator (the pair rounded to FP64): residuals at the FP64 floor
    z = lambda c: (c[0] + c[1]) + 1j * (c[2] + c[3])  # noqa: E731
    v3 = verify_pair(z(a), SchurPair(q=z(qc), t=z(pair.t.to_numpy_cells()), ortho_residual=0.0), precision="fp64")
    u64 = 2.0 ** -53
    assert v3.tri_residual <= 10 * n * u64 * norm_a and v3.ortho_residual <= 10 * n * u64
