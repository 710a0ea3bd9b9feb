"""ORACLE — test infrastructure only.

CPU restatement of the reference's `refine_template` loop in the FP64 mode
the BASELINE configs ask for (hp = complex128, lp = complex64).  The
reference itself only runs hp = double-double / lp = binary64; this module
keeps its control flow line for line and swaps the two precisions:

  refine_template        /root/reference/pkg/src/ddschur/refine.py:357-380
  _run (the loop)        refine.py:223-329
  status / skip / streak refine.py:269-321
  newton_schulz_step     /root/reference/pkg/src/ddschur/orthogonal.py:153-169
  spectral_norm_estimate /root/reference/pkg/src/ddschur/matmul.py:117-142
  merged_update          orthogonal.py:172-201
  solve_block            trisolve.py:243-262 via oracle/trisolve_oracle.c
                         in complex64 arithmetic

hp products are numpy complex128 matmuls (BLAS), lp products complex64.
Row 0 of the history: the reference measures it in lp right after the entry
orthogonalisation (refine.py:126-135,237).  In FP64 mode lp is complex64,
whose noise (~1e-7) swamps the entry residual, so — as SURVEY.md §8a6
recommends — row 0 is measured in FP64 (hp).  Iteration 1 measures the same
Q in the same precision, so row 0 equals row 1 exactly; the GPU product
shares that measurement instead of repeating three GEMMs.
"""
import math
import time

import numpy as np

from . import clib

U_FP64 = 2.0 ** -53


def spectral_norm_estimate(m, rel_tol=1e-6, max_iters=200):
    """matmul.py:117-142, power iteration on M^H M in lp (complex64)."""
    m = np.asarray(m, dtype=np.complex64)
    cols = m.shape[1]
    v = (1.0 + (np.arange(cols) % 7) / 8.0).astype(np.complex64)
    v = v / np.linalg.norm(v)
    prev = 0.0
    est = 0.0
    for _ in range(max_iters):
        u = m @ v
        est = float(np.linalg.norm(u))
        if est == 0.0:
            return 0.0
        w = m.conj().T @ u
        nw = float(np.linalg.norm(w))
        if nw == 0.0:
            return est
        v = w / nw
        if abs(est - prev) <= rel_tol * est:
            break
        prev = est
    return est


def newton_schulz_step(qhat):
    """orthogonal.py:153-169 with hp = complex128."""
    est = spectral_norm_estimate(qhat)
    if not est < math.sqrt(3.0):
        raise ValueError("NormTooLarge: spectral norm estimate %.6f" % est)
    n = qhat.shape[0]
    g = qhat.conj().T @ qhat
    sigma = 3.0 * np.eye(n) - g
    return 0.5 * (qhat @ sigma)


def merged_update(q, w, y, restore_full_sigma=False):
    """orthogonal.py:172-201: products of the small factors in lp
    (complex64), the Sigma sum in hp left to right, one hp product.

    W is scaled by a power of two 2^-k (exact) to unit size before its lp
    products and the products are scaled back after the upcast: the same
    values bit for bit whenever the unscaled products stay in complex64's
    normal range, and no subnormal W^3 (|W| ~ 1e-12 near convergence gives
    |W^3| ~ 1e-36), on which x86 BLAS takes a ~100x slower microcode path."""
    n = q.shape[0]
    y_lp = y.astype(np.complex64)
    w = w.astype(np.complex64)
    nw = float(np.max(np.abs(w))) if w.size else 0.0
    k = int(np.frexp(nw)[1]) if nw > 0.0 else 0
    ws = np.ldexp(w.real, -k) + 1j * np.ldexp(w.imag, -k)
    ws = ws.astype(np.complex64)

    def up(x, e):  # complex64 product of scaled factors -> complex128, times 2^e (exact)
        x = x.astype(np.complex128)
        return np.ldexp(x.real, e) + 1j * np.ldexp(x.imag, e)
    yw_s = y_lp @ ws
    w2_s = ws @ ws
    w3_s = w2_s @ ws
    sigma = 2.0 * np.eye(n, dtype=np.complex128) + (2.0 * w).astype(np.complex128)
    sigma = sigma - y
    sigma = sigma - up(yw_s, k)
    sigma = sigma + up(w2_s, 2 * k)
    sigma = sigma + up(w3_s, 3 * k)
    if restore_full_sigma:
        w2y_s = w2_s @ y_lp
        w2yw_s = w2y_s @ ws
        sigma = sigma + up(w2y_s, 2 * k)
        sigma = sigma + up(w2yw_s, 3 * k)
    return 0.5 * (q @ sigma)


def refine_template_fp64(a, qhat, tol_factor=10.0, max_iters=20, n_min=4,
                         clip_threshold=None, skip_final_ortho=True,
                         restore_full_sigma=False, solver="c"):
    """refine.py:357-380 + _run (223-329) in FP64 mode.  Returns a dict.

    solver "c": the plain-C restatement of trisolve.py (the parity checker);
    "blas": oracle/trisolve_blas.py, the same recursion on BLAS / LAPACK
    kernels (the timed CPU baseline at large n; no clipping)."""
    if solver not in ("c", "blas"):
        raise ValueError("solver must be 'c' or 'blas'")
    if solver == "blas" and clip_threshold is not None:
        raise ValueError("the BLAS solver port does not clip")
    t0 = time.perf_counter()
    a = np.asarray(a)
    a = a.astype(np.complex128) if np.iscomplexobj(a) else a.astype(np.float64)
    qhat = np.ascontiguousarray(qhat, dtype=np.complex128)
    n = a.shape[0]
    if a.shape != (n, n) or qhat.shape != (n, n):
        raise ValueError("refinement needs square matrices of equal shape")
    if not (np.isfinite(a).all() and np.isfinite(qhat).all()):
        raise ValueError("input matrix has non-finite entries")
    hp = 0
    phases = dict(entry=0.0, measure=0.0, solve=0.0, update=0.0)
    tp = time.perf_counter()
    q = newton_schulz_step(qhat)
    hp += 2
    phases["entry"] += time.perf_counter() - tp
    norm_a = float(np.linalg.norm(a))
    tol = tol_factor * n * U_FP64 * norm_a
    history = []
    clipped_total = 0
    skip_fired = False
    detail = ""
    status = "MaxIters"
    iterations = max_iters
    that = None
    streak = 0
    eye = np.eye(n)
    real_a = not np.iscomplexobj(a)
    for it in range(1, max_iters + 1):
        tp = time.perf_counter()
        if real_a:  # Q^H A with real A: two real products (the same values up to rounding)
            qha = (q.real.T @ a) - 1j * (q.imag.T @ a)
        else:
            qha = q.conj().T @ a
        that = qha @ q
        del qha
        hp += 2
        e = np.tril(that, -1)
        t = np.triu(that)
        norm_e = float(np.linalg.norm(e))
        y = q.conj().T @ q - eye
        hp += 1
        norm_y = float(np.linalg.norm(y))
        phases["measure"] += time.perf_counter() - tp
        if it == 1:
            history.append((norm_e, norm_y))  # row 0: FP64 entry measurement
        history.append((norm_e, norm_y))
        if not (math.isfinite(norm_e) and math.isfinite(norm_y)):
            status, iterations = "NonFinite", it
            detail = "iteration %d: residuals became non-finite" % it
            break
        converged = norm_e <= tol
        tp = time.perf_counter()
        try:
            if solver == "c":
                l, nclip = clib.solve_block(t.astype(np.complex64), e.astype(np.complex64),
                                            n_min=n_min, clip_threshold=clip_threshold,
                                            dtype=np.complex64)
            else:
                from . import trisolve_blas
                l, nclip = trisolve_blas.solve_block(t, e, n_min=n_min, dtype=np.complex64), 0
        except clib.NonFiniteError as exc:
            status, iterations = "NonFinite", it
            detail = "iteration %d: %s" % (it, exc)
            break
        clipped_total += nclip
        w = l - l.conj().T
        norm_w = float(np.linalg.norm(w))
        phases["solve"] += time.perf_counter() - tp
        skip = (converged and skip_final_ortho and norm_y <= 10.0 * n * U_FP64
                and norm_w <= math.sqrt(U_FP64))
        if not skip:
            tp = time.perf_counter()
            q = merged_update(q, w, y, restore_full_sigma)
            hp += 1
            phases["update"] += time.perf_counter() - tp
        if converged:
            status, iterations, skip_fired = "Converged", it, skip
            break
        if len(history) >= 2 and norm_e > history[-2][0]:
            streak += 1
        else:
            streak = 0
        if streak >= 3:
            status, iterations = "Diverged", it
            break
    last_e, last_y = history[-1]
    return dict(q=q, t=np.triu(that), ortho_residual=last_y, tri_residual=last_e,
                iterations=iterations, residual_history=history, hp_matmul_count=hp,
                clipped_total=clipped_total, status=status, skip_fired=skip_fired,
                detail=detail, wall_time=time.perf_counter() - t0, norm_a=norm_a, phases=phases)


def residuals_fp64(a, q):
    """FP64 evaluator of the three parity quantities (verify_pair's first
    two, refine.py:456-476, in complex128): (relE, ||Q^H Q - I||_F)."""
    a = np.asarray(a)
    q = np.asarray(q, dtype=np.complex128)
    that = (q.conj().T @ a) @ q
    rel_e = float(np.linalg.norm(np.tril(that, -1)) / np.linalg.norm(a))
    ortho = float(np.linalg.norm(q.conj().T @ q - np.eye(q.shape[0])))
    return rel_e, ortho
