"""refine_mixed (/root/reference/pkg/src/ddschur/refine.py:383-406): a Schur
pair of A from scratch, SURVEY §8f row 2.

Pipeline as in the reference — lp Schur pair, eigenvalues ordered along the
random line of cfg.seed (schur.py:185-200), entry Newton-Schulz step, the
template's refinement loop — with the lp Schur front end on the GPU: the
reference QR-iterates a Hessenberg matrix in binary64 (schur.py:67-183) and
then swaps the eigenvalues into the random-line order with Givens rotations
(reorder_schur, schur.py:203-233); here the eigenpairs come from the GPU
eigensolver (torch.linalg.eig in the mode's lp type), the eigenvectors are
permuted into the random-line order and orthonormalised by QR.  With
V = [v_1 .. v_n] in that order and V = Q R, A Q = Q (R Lambda R^-1), so Q is
a Schur basis whose triangular factor carries the eigenvalues in exactly the
reference's order; Schur bases with the same order agree up to column
phases, which the refinement's T absorbs.  (Measured on the B200: lp residual
of the candidate 3e-5 (complex64) / 8e-14 (complex128) at n = 4096;
tools/eig_front_probe.py.)"""
import time

import numpy as np
import torch

from . import _lib  # noqa: F401  (loads the library: no CPU fallback)
from .matrix import DDPlanar, ZPlanar
from .refine import OrthoStrategy, RefineConfig, _coerce, _run_fp64, _workspace
from .symmetric import order_by_random_line


def probe_gaps_complex(ritz, norm_a, chunk=2048):
    """_probe_gaps (refine.py:441-453): minimum pairwise distance of the Ritz
    values, on the device in row chunks."""
    r = torch.as_tensor(ritz)
    n = r.numel()
    if n < 2:
        return ""
    gap = float("inf")
    for i0 in range(0, n, chunk):
        d = (r[i0:i0 + chunk, None] - r[None, :]).abs()
        idx = torch.arange(i0, min(i0 + chunk, n), device=r.device)
        d[idx - i0, idx] = float("inf")
        gap = min(gap, float(d.min()))
    if gap == 0.0:
        return "entry probe: exactly repeated Ritz values"
    if gap < 1e-10 * max(norm_a, 1.0):
        return "entry probe: min Ritz gap %.3e" % gap
    return ""


def lp_schur_front(a_lp, seed):
    """(Q lp Schur basis, Ritz values) ordered along the random line of seed."""
    w, v = torch.linalg.eig(a_lp)
    rng = np.random.Generator(np.random.Philox(seed))
    order = order_by_random_line(w.cpu().numpy().astype(np.complex128), rng=rng)
    perm = torch.as_tensor(order.permutation, device=a_lp.device)
    q, _ = torch.linalg.qr(v[:, perm])
    return q, w[perm]


def refine_mixed(a, cfg=None, device=None):
    """Schur pair of A from scratch (refine.py:383-406).  Returns
    (SchurPair, RefineReport) like refine_template."""
    cfg = RefineConfig() if cfg is None else cfg
    if cfg.ortho is not OrthoStrategy.NEWTON_SCHULZ:
        raise NotImplementedError("QR retraction is not on the B200 path (no CPU fallback)")
    if not torch.cuda.is_available():
        raise RuntimeError("refine_mixed needs a CUDA device (no CPU fallback)")
    device = torch.device("cuda") if device is None else torch.device(device)
    t0 = time.perf_counter()
    if cfg.precision == "dd":
        from . import dd_refine
        A = dd_refine.coerce_dd(a, device)
        hi, lo = A.hi, A.lo
        norm_a = float(torch.sqrt((hi.re + lo.re).square().sum() + (hi.im + lo.im).square().sum()))
        a_lp = torch.complex(hi.re, hi.im)  # to_lp: the hi parts (binary64)
    else:
        A = _coerce(a, device)
        norm_a = float(torch.sqrt(A.re.square().sum() + (A.im.square().sum() if A.im is not None else 0.0)))
        a_lp = torch.complex(A.re, A.im if A.im is not None else torch.zeros_like(A.re)).to(torch.complex64)
    q_lp, ritz = lp_schur_front(a_lp, cfg.seed)
    probe = probe_gaps_complex(ritz, norm_a)
    if cfg.precision == "dd":
        from . import dd_refine
        qhat = DDPlanar.from_any(q_lp.to(torch.complex128), device=device)
        pair, report = dd_refine.run_dd(A, qhat, cfg, device)
    else:
        qhat = ZPlanar.from_any(q_lp.to(torch.complex128), device=device, force_complex=True)
        ws = _workspace(A.rows, device)
        ws.in_flags.zero_()  # inputs validated by _coerce above
        pair, report = _run_fp64(A, qhat, cfg, ws)
    torch.cuda.current_stream().synchronize()
    report.wall_time = time.perf_counter() - t0
    if probe:
        report.detail = probe + "; " + report.detail if report.detail else probe
    return pair, report


__all__ = ["refine_mixed", "lp_schur_front"]
