"""The reference's orthogonalisation boundary (ddschur.orthogonal) on the B200.

  newton_schulz_step  /root/reference/pkg/src/ddschur/orthogonal.py:153-169
  merged_update       orthogonal.py:172-201
  NormTooLarge        orthogonal.py:38

Both run the refinement's own product kernels (Ozaki-II on the int8 tensor
cores): a double-double operand (DDMatrix, DDPlanar, anything with
`.cells()`) runs in the reference's dd mode (hp = dd, lp = binary64) and
returns the same kind; an FP64 operand (ZPlanar, a complex numpy / torch
matrix) runs in FP64 mode (hp = FP64, lp = complex64) and returns a complex128
CUDA tensor.  The products are formed as in the refinement loop:
Q^ (3I - G) / 2 = Q^ - Q^ (G - I) / 2 and Q Sigma / 2 = Q + Q (Sigma - 2I) / 2
— the same matrices as the reference's, with one rounding at the end — and
each call counts its hp products in the reference's counters (2 and 1).
"""
import math

import numpy as np
import torch

from . import _lib
from .ddmatrix import DDMatrix, _is_dd, as_ddplanar
from .errors import NormTooLarge
from .matmul import spectral_norm_estimate
from .matrix import DDPlanar, ZPlanar


def _stream():
    return torch.cuda.current_stream().cuda_stream


def _guard(hi, n, ws_c64):
    """||Q^||_2 < sqrt(3) by lp power iteration (orthogonal.py:160-166)."""
    _lib.call("sr_downcast_c64", n, n, hi.re_ptr(), hi.im_ptr(), hi.ld, ws_c64.data_ptr(), ws_c64.shape[1],
              _stream())
    est = spectral_norm_estimate(ws_c64, n)
    if not est < math.sqrt(3.0):
        raise NormTooLarge("spectral norm estimate %.6f is not below sqrt(3)" % est)


def _dd_products(n, device):
    from . import dd_refine
    ws = dd_refine._workspace(n, device)
    return ws, dd_refine.DDProducts(ws, None)


def _fp64_products(n, device, gauss=True):
    from . import products, refine
    ws = refine._workspace(n, device)
    return ws, products.OzakiProducts(ws, None, gauss=gauss)


def _is_skew(w):
    """W exactly skew-Hermitian (as W = L - L^H always is in floating point)."""
    return bool(torch.equal(w, -w.mH))


def _result_dd(x, host):
    out = DDPlanar.empty(x.rows, x.cols, device=x.hi.re_buf.device)
    out.hi.copy_(x.hi)
    out.lo.copy_(x.lo)
    return out.to_ddmatrix() if host else out


def newton_schulz_step(qhat, device=None):
    """One Newton-Schulz step Q = Q^ (3I - Q^H Q^) / 2 (orthogonal.py:153-169):
    exactly two hp products; NormTooLarge unless ||Q^||_2 < sqrt(3)."""
    device = torch.device("cuda") if device is None else torch.device(device)
    if _is_dd(qhat):
        host = not isinstance(qhat, DDPlanar)
        q = as_ddplanar(qhat, device=device)
        n = q.rows
        if q.cols != n:
            raise ValueError("newton_schulz_step expects a square matrix")
        ws, prod = _dd_products(n, device)
        _guard(q.hi, n, ws.q_c64)
        prod.entry(q)
        return _result_dd(ws.q, host)
    q = ZPlanar.from_any(qhat, device=device, force_complex=True)
    n = q.rows
    if q.cols != n:
        raise ValueError("newton_schulz_step expects a square matrix")
    ws, prod = _fp64_products(n, device)
    _guard(q, n, ws.y_lp)
    prod.entry(q)  # counts its two hp products
    return ws.q.to_complex()


def merged_update(q, w, y, restore_full_sigma=False, device=None):
    """Newton-Schulz step on Q(I + W) merged into one hp product
    (orthogonal.py:172-201): Q_new = Q Sigma / 2 with
    Sigma = 2I + 2W - Y - YW + W^2 + W^3 (+ W^2 Y + W^2 Y W), the products of
    the small factors in lp, the sum in hp left to right.  q, y: hp (y =
    Q^H Q - I); w: the lp correction (n x n)."""
    device = torch.device("cuda") if device is None else torch.device(device)
    if _is_dd(q):
        host = not isinstance(q, DDPlanar)
        Q = as_ddplanar(q, device=device)
        Y = as_ddplanar(y, device=device)
        n = Q.rows
        W = torch.as_tensor(np.asarray(w) if not torch.is_tensor(w) else w)
        if Q.cols != n or tuple(W.shape) != (n, n) or Y.shape != (n, n):
            raise ValueError("q, w, y must all be n x n")
        ws, prod = _dd_products(n, device)
        Wd = W.to(device=device, dtype=torch.complex128)
        prod.w_skew = _is_skew(Wd)
        ws.q.hi.copy_(Q.hi)
        ws.q.lo.copy_(Q.lo)
        ws.y.hi.copy_(Y.hi)
        ws.y.lo.copy_(Y.lo)
        ws.w_lp[:, :n].copy_(Wd)
        prod.update(restore_full_sigma)
        return _result_dd(ws.q, host)
    Q = ZPlanar.from_any(q, device=device, force_complex=True)
    Y = ZPlanar.from_any(y, device=device, force_complex=True)
    n = Q.rows
    W = torch.as_tensor(np.asarray(w) if not torch.is_tensor(w) else w)
    if Q.cols != n or tuple(W.shape) != (n, n) or Y.shape != (n, n):
        raise ValueError("q, w, y must all be n x n")
    from . import products
    Wd = W.to(device=device, dtype=torch.complex64)
    skew = _is_skew(Wd)
    # the Gaussian planes' single encoding of W needs W skew-Hermitian
    ws, prod = _fp64_products(n, device, gauss=skew)
    prod.w_skew = skew
    ws.q.copy_(Q)
    ws.y.copy_(Y)
    ws.w_lp[:, :n].copy_(Wd)
    if restore_full_sigma:
        products.ensure_full_sigma_buffers(ws)
    prod.update(restore_full_sigma)
    return ws.q.to_complex()


__all__ = ["NormTooLarge", "merged_update", "newton_schulz_step", "DDMatrix"]
