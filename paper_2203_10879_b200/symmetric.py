"""refine_symmetric (/root/reference/pkg/src/ddschur/refine.py:409-438): the
Hermitian variant of the refinement, SURVEY §8f row 3.

For Hermitian A the converged T is diagonal, so the lp solve collapses to
the entrywise l_ij = -e_ij / (t_ii - t_jj) (csrc/elementwise.cu,
sr_diag_correction_*) and the defect is the full off-diagonal part of
Q^H A Q; everything else is the template's loop (refine._run_fp64 /
dd_refine.run_dd with symmetric=True) on the same tensor-core products.

The lp front end replaces the reference's binary64 QR iteration
(schur.qr_schur_lp) by the Hermitian eigensolver (cuSOLVER heevd through
torch.linalg.eigh, in the mode's lp type): for Hermitian A the Schur
vectors are eigenvectors, and after the same random-line ordering
(schur.py:185-200, Philox(cfg.seed)) the candidate matches the reference's
up to column phases, which the refinement does not see in T."""
import dataclasses
import time

import numpy as np
import torch

from . import _lib  # noqa: F401  (loads the library: no CPU fallback)
from .errors import NotSymmetric
from .matrix import DDPlanar, ZPlanar
from .refine import U_FP64, U_HP, OrthoStrategy, RefineConfig, _coerce, _run_fp64, _workspace


@dataclasses.dataclass
class EigOrder:
    """schur.py:53-55."""

    permutation: np.ndarray


def order_by_random_line(eigs, rng=None, theta=None):
    """order_by_random_line (schur.py:185-200): stable sort of the eigenvalues
    projected on a random line through the origin, direction from rng."""
    eigs = np.asarray(eigs, dtype=complex)
    if eigs.ndim != 1 or eigs.size < 1:
        raise ValueError("need a 1-d nonempty eigenvalue array")
    if theta is None:
        if rng is None:
            rng = np.random.Generator(np.random.Philox(0))
        theta = float(rng.uniform(0.0, 2.0 * np.pi))
    keys = np.real(np.exp(-1j * theta) * eigs)
    return EigOrder(permutation=np.argsort(keys, kind="stable"))


def probe_gaps(ritz, norm_a):
    """_probe_gaps (refine.py:441-453) for real Ritz values (sorted neighbours
    give the minimum pairwise gap)."""
    r = np.sort(np.asarray(ritz, dtype=float))
    if r.size < 2:
        return ""
    gap = float(np.min(np.diff(r)))
    if gap == 0.0:
        return "entry probe: exactly repeated Ritz values"
    if gap < 1e-10 * max(norm_a, 1.0):
        return "entry probe: min Ritz gap %.3e" % gap
    return ""


def _defect_planes(re, im):
    """||X - X^H||_F^2 of planar (re, im): re antisymmetric part, im symmetric part."""
    d = (re - re.T).square().sum()
    if im is not None:
        d = d + (im + im.T).square().sum()
    return d


def refine_symmetric(a, cfg=None, device=None):
    """Hermitian-input refinement from scratch (refine.py:409-438).  Raises
    NotSymmetric unless ||A - A^H||_F <= 10 u_hp ||A||_F.  Returns
    (SchurPair, RefineReport) like refine_template; T has real entries."""
    cfg = RefineConfig() if cfg is None else cfg
    if cfg.ortho is not OrthoStrategy.NEWTON_SCHULZ:
        raise NotImplementedError("QR retraction is not on the B200 path (no CPU fallback)")
    if not torch.cuda.is_available():
        raise RuntimeError("refine_symmetric needs a CUDA device (no CPU fallback)")
    device = torch.device("cuda") if device is None else torch.device(device)
    t0 = time.perf_counter()
    if cfg.precision == "dd":
        from . import dd_refine
        A = dd_refine.coerce_dd(a, device)
        u = U_HP
        hi, lo = A.hi, A.lo
        norm_a = float(torch.sqrt(sum((c.square().sum() for c in (hi.re + lo.re, hi.im + lo.im)))))
        # the hi parts cancel exactly for a Hermitian dd matrix; add the lo parts' defect
        dr = (hi.re - hi.re.T) + (lo.re - lo.re.T)
        di = (hi.im + hi.im.T) + (lo.im + lo.im.T)
        defect = float(torch.sqrt(dr.square().sum() + di.square().sum()))
        a_lp = torch.complex(hi.re, hi.im)  # to_lp: the hi parts (binary64)
    else:
        A = _coerce(a, device)
        u = U_FP64
        norm_a = float(torch.sqrt(A.re.square().sum() + (A.im.square().sum() if A.im is not None else 0.0)))
        defect = float(torch.sqrt(_defect_planes(A.re, A.im)))
        a_lp = torch.complex(A.re, A.im if A.im is not None else torch.zeros_like(A.re)).to(torch.complex64)
    if defect > 10.0 * u * norm_a:
        raise NotSymmetric("||A - A^H||_F = %.3e exceeds 10 u_hp ||A||_F = %.3e" % (defect, 10.0 * u * norm_a))
    # lp front end: eigenpairs, ordered along the random line of cfg.seed
    a_lp = (a_lp + a_lp.conj().T) / 2  # exactly Hermitian for the eigensolver
    w, v = torch.linalg.eigh(a_lp)
    rng = np.random.Generator(np.random.Philox(cfg.seed))
    order = order_by_random_line(w.double().cpu().numpy(), rng=rng)
    perm = torch.as_tensor(order.permutation, device=device)
    v = v[:, perm]
    probe = probe_gaps(w.double().cpu().numpy()[order.permutation], norm_a)
    if cfg.precision == "dd":
        from . import dd_refine
        qhat = DDPlanar.from_any(v.to(torch.complex128), device=device)
        pair, report = dd_refine.run_dd(A, qhat, cfg, device, symmetric=True)
    else:
        qhat = ZPlanar.from_any(v.to(torch.complex128), device=device, force_complex=True)
        ws = _workspace(A.rows, device)
        ws.in_flags.zero_()  # inputs validated by _coerce above
        pair, report = _run_fp64(A, qhat, cfg, ws, symmetric=True)
    torch.cuda.current_stream().synchronize()
    report.wall_time = time.perf_counter() - t0
    if probe:
        report.detail = probe + "; " + report.detail if report.detail else probe
    return pair, report


__all__ = ["refine_symmetric", "order_by_random_line", "EigOrder", "probe_gaps"]
