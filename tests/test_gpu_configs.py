"""Parity at the BASELINE configs' STATED sizes (VERDICT r1, rows C2–C5).

  C2  n = 2048 complex Gaussian, complex64-Schur start, FP64 mode: against the
      CPU restatement run in-test on the same inputs (C solver), its committed
      golden run (tests/golden/oracle_config2.json) and the unmodified
      reference's own run (tests/golden/config2_ref.json, dd hp, FP64 stop).
  C3  n = 8192 real Gaussian (the bench workload): the refined pair is
      re-evaluated by two evaluators independent of the refinement's own
      measurement — verify_pair in double-double (Ozaki-II at beta = 106,
      dd intermediates) and a cuBLAS ZGEMM evaluation (test-only) — and the
      run is compared with the committed CPU-restatement golden
      (tests/golden/oracle_config3.json: status, iterations ±1, entry residual).
  C4  n = 1024 dd mode: the literal matrix (the reference ends NonFinite at
      iteration 3) and the well-conditioned variant (reference: Converged in
      3, verify 1.1e-30 / 1.8e-30) against tests/golden/configs_full_ref.json.
  C5  the full 64-step n = 512 continuation chain against the committed
      oracle chain (tests/golden/oracle_config5.json).

Tolerances: same status, iterations ±1, relE <= 10 u64 (FP64
mode), ||Q^H Q - I||_F within 2x of the restatement's (same evaluator);
dd mode: ortho <= 1e-28 and tri <= 10 n 2^-106 ||A||_F (test_acceptance.py:48-49).

The Q̂ matrices are LAPACK cgees / zgees outputs rebuilt here with the same
call as the golden generators (16–512 MiB, not committed); each golden case
records the digest of its Q̂, and the history comparisons that depend on the
exact bits of Q̂ only run when the digests agree.
"""
import hashlib
import json
import os

import numpy as np
import pytest
import torch

from oracle.refine_fp64 import refine_template_fp64, residuals_fp64
from paper_2203_10879_b200 import RefineConfig, RefineStatus, SchurPair, ZPlanar, inputs, refine_template, verify_pair

pytestmark = pytest.mark.gpu
U = 2.0 ** -53
U_HP = 2.0 ** -106
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def golden_cases(name):
    with open(os.path.join(GOLDEN, name + ".json")) as f:
        return json.load(f)["cases"]


def digest(x):
    return hashlib.sha256(np.ascontiguousarray(x).tobytes()).hexdigest()[:16]


def fp64_cfg(n, **kw):
    return RefineConfig(precision="fp64", tol_factor=10.0 / n, max_iters=10, **kw)


def test_config2_n2048_matches_oracles():
    a, q = inputs.config_inputs(2)
    n = a.shape[0]
    assert n == 2048
    pair, rep = refine_template(a, q, fp64_cfg(n))
    ref = refine_template_fp64(a, q, tol_factor=10.0 / n, max_iters=10)
    assert rep.status.value == ref["status"] == "Converged", (rep.status, ref["status"])
    assert abs(rep.iterations - ref["iterations"]) <= 1
    assert rep.hp_matmul_count == 2 + 4 * rep.iterations - (1 if rep.skip_fired else 0)
    rel_e, ortho = residuals_fp64(a, pair.q.cpu().numpy())
    _, ortho_o = residuals_fp64(a, ref["q"])
    assert rep.residual_history[-1][0] / ref["norm_a"] <= 10 * U
    assert rel_e <= 10 * U, rel_e
    assert ortho <= 2 * ortho_o, (ortho, ortho_o)
    # the entry residual: the same FP64 state measured by both
    assert np.isclose(rep.residual_history[0][0], ref["residual_history"][0][0], rtol=1e-6)
    g = golden_cases("oracle_config2")[0]
    assert rep.status.value == g["status"] and abs(rep.iterations - g["iterations"]) <= 1
    if digest(q.astype(np.complex64)) == g["qhat_sha256_16"] or digest(q) == g["qhat_sha256_16"]:
        assert np.isclose(rep.residual_history[0][0], g["residual_history"][0][0], rtol=1e-6)
    path = os.path.join(GOLDEN, "config2_ref.json")
    if os.path.exists(path):  # the unmodified reference (dd hp) with the FP64 stop rule
        r = golden_cases("config2_ref")[0]
        assert rep.status.value == r["status"] and abs(rep.iterations - r["iterations"]) <= 1, r


def test_config3_n8192_independent_evaluation():
    a, q = inputs.config_inputs(3)
    n = a.shape[0]
    assert n == 8192
    dev = torch.device("cuda")
    A, Qh = ZPlanar.from_any(a, device=dev), ZPlanar.from_any(q, device=dev)
    pair, rep = refine_template(A, Qh, fp64_cfg(n))
    norm_a = float(np.linalg.norm(a))
    g = golden_cases("oracle_config3")[0]
    assert rep.status.value == g["status"] == "Converged", (rep.status, g["status"])
    assert abs(rep.iterations - g["iterations"]) <= 1, (rep.iterations, g["iterations"])
    assert rep.hp_matmul_count == 2 + 4 * rep.iterations - (1 if rep.skip_fired else 0)
    if digest(q.astype(np.complex64)) == g["qhat_sha256_16"]:
        # same Q̂ bits: the entry residual (FP64 entry step, then an exact
        # measurement here / a BLAS one in the restatement) agrees
        assert np.isclose(rep.residual_history[0][0], g["residual_history"][0][0], rtol=1e-4)
    own_rel_e, own_ortho = rep.residual_history[-1][0] / norm_a, rep.residual_history[-1][1]
    assert own_rel_e <= 10 * U
    # (1) verify_pair in double-double: P = Q^H A and T^ = P Q kept in dd
    v = verify_pair(A, SchurPair(q=pair.q, t=pair.t, ortho_residual=0.0), precision="dd")
    assert v.tri_residual / norm_a <= 10 * U, v
    # the refinement's own ||Y|| (FP64-rounded entries of an exact product of the
    # beta-truncated Q) agrees with the dd evaluation to a few digits
    assert abs(v.ortho_residual - own_ortho) <= 1e-2 * own_ortho, (v.ortho_residual, own_ortho)
    assert v.similarity_residual / norm_a <= 10 * U, v
    assert own_ortho <= 2 * g["final_ortho"], (own_ortho, g["final_ortho"])
    # (2) cuBLAS ZGEMM (FP64, test-only): its own accumulation noise on
    # stril(Q^H A Q) is ~20 u ||A||_F at n = 8192 (measured 2.4e-15 — above
    # the 10 u stop rule, the reason the products are exact Ozaki-II ones,
    # DESIGN.md §3.1), so it confirms the residual only to that noise floor
    qd = pair.q
    ad = torch.from_numpy(a).to(dev).to(torch.complex128)
    that = (qd.conj().T @ ad) @ qd
    rel_z = float(torch.linalg.norm(torch.tril(that, -1))) / norm_a
    ortho_z = float(torch.linalg.norm(qd.conj().T @ qd - torch.eye(n, dtype=torch.complex128, device=dev)))
    del that, ad
    assert rel_z <= 50 * U, rel_z
    assert ortho_z <= n * U, (ortho_z, g["final_ortho"])  # cuBLAS FP64 Gram noise (3.6e-13 measured)


@pytest.mark.parametrize("tag", ["config4_n1024", "config4wc_n1024"])
def test_config4_n1024_dd_matches_reference(tag):
    c = [c for c in golden_cases("configs_full_ref") if c["tag"] == tag][0]
    n = c["n"]
    scale = 1.0 / np.sqrt(n) if tag.startswith("config4wc") else 1.0
    a = inputs.config4_matrix(n, 0, strict_scale=scale)
    q = inputs.schur_vectors(a, np.complex128)
    pair, rep = refine_template(a, q, RefineConfig(precision="dd", max_iters=10))
    assert rep.status.value == c["status"], (tag, rep.status, c["status"], rep.detail)
    assert abs(rep.iterations - c["iterations"]) <= 1, (tag, rep.iterations, c["iterations"])
    if digest(q) == c["qhat_sha256_16"]:  # same Q̂ bits: the binary64 entry measurement agrees
        assert np.isclose(rep.residual_history[0][0], c["residual_history"][0][0], rtol=1e-3)
    if rep.status is RefineStatus.NON_FINITE:
        assert rep.detail.startswith("iteration %d:" % rep.iterations)
        return
    norm_a = np.linalg.norm(a)
    v = verify_pair(a, pair, precision="dd")
    assert v.ortho_residual <= 1e-28, v
    assert v.tri_residual <= 10 * n * U_HP * norm_a, v
    # the reference's own verify_pair of its result: the same dd noise floor
    ro, rt, _ = c["verify"]
    assert v.ortho_residual <= 10 * ro and v.tri_residual <= 10 * rt, (v, c["verify"])


def test_config5_full_chain_matches_oracle_chain():
    """64 steps of n = 512: A(t_j) = A0 + t_j A1, t_j = 0.01 j / 64, each
    step from the previous refined Q (refine_continuation)."""
    from paper_2203_10879_b200 import refine_continuation
    g = golden_cases("oracle_config5")[0]
    n, steps = g["n"], g["steps"]
    a0, a1 = inputs.config5_pair(n, 0)
    q0 = inputs.schur_vectors(a0).astype(np.complex128)
    ts = [0.01 * j / 64 for j in range(steps)]
    chain = refine_continuation(a0, a1, ts, q0, fp64_cfg(n))
    assert len(chain) == steps == len(g["chain"])
    for (t, pair, rep), gc in zip(chain, g["chain"]):
        a = a0 + t * a1
        assert rep.status.value == gc["status"] == "Converged", (t, rep.status, gc)
        assert abs(rep.iterations - gc["iterations"]) <= 1, (t, rep.iterations, gc["iterations"])
        rel_e, ortho = residuals_fp64(a, pair.q.cpu().numpy())
        assert rel_e <= 10 * U * 1.5, (t, rel_e)
        assert ortho <= 2 * max(gc["final_ortho"], 10 * np.sqrt(n) * U), (t, ortho, gc["final_ortho"])
