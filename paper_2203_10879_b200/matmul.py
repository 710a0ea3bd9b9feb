"""hp / lp matrix products on the B200 (FP64 mode), reference-named.

  matmul_hp               /root/reference/pkg/src/ddschur/matmul.py:52-81
  matmul_lp               matmul.py:84-110
  spectral_norm_estimate  matmul.py:117-142
  counters/reset_counters matmul.py:33-42 (logical products, not launches)

Both products run through libsr.so (sr_zgemm_f64 on the FP64 DMMA pipe,
sr_cgemm_c64 on the FP32 pipe); the counters count logical products the
way the reference does, and `hp_seconds` / `lp_seconds` are left at zero
because device work is asynchronous (time it with CUDA events instead).
"""
import torch

from . import _lib
from .matrix import ZPlanar, lp_empty

_counters = {"hp_calls": 0, "hp_seconds": 0.0, "lp_calls": 0, "lp_seconds": 0.0}


def reset_counters():
    for k in _counters:
        _counters[k] = 0.0 if k.endswith("seconds") else 0


def counters():
    return dict(_counters)


def _stream():
    return ctypes_stream(torch.cuda.current_stream())


def ctypes_stream(s):
    return s.cuda_stream


DD_PRODUCT_BETA = 106  # standalone dd products: every entry within 2^0 of its row max keeps 106 bits


def _matmul_dd(a, b, trans_a, trans_b):
    """C = op(A) op(B) in double-double (the reference's matmul_hp on
    DDMatrix operands, matmul.py:52-81): an Ozaki-II product with dd in and
    out (csrc/ozaki.cu, SR_MAT_DD); op(B) = B^H materialised on the device
    first, like the reference (matmul.py:64-65).  Host DDMatrix operands give
    a host DDMatrix, device DDPlanar ones a DDPlanar."""
    from . import ozaki
    from .ddmatrix import as_ddplanar
    from .matrix import DDPlanar
    host = not (isinstance(a, DDPlanar) and isinstance(b, DDPlanar))
    A = as_ddplanar(a)
    B = as_ddplanar(b, device=A.hi.re_buf.device)
    if trans_b:
        dev = B.hi.re_buf.device
        Bt = DDPlanar.empty(B.cols, B.rows, device=dev)
        for src, dst, sgn in ((B.hi.re, Bt.hi.re_buf, 1.0), (B.lo.re, Bt.lo.re_buf, 1.0),
                              (B.hi.im, Bt.hi.im_buf, -1.0), (B.lo.im, Bt.lo.im_buf, -1.0)):
            dst[:, : B.rows].copy_(src.t() * sgn if sgn < 0 else src.t())
            dst[:, B.rows:].zero_()
        B = Bt
    m, k = (A.cols, A.rows) if trans_a else (A.rows, A.cols)
    if B.rows != k:
        raise ValueError("inner dimensions disagree: %d vs %d" % (k, B.rows))
    n = B.cols
    pl = ozaki.plan(max(k, 1), DD_PRODUCT_BETA, DD_PRODUCT_BETA)
    ea = ozaki.encode(A, A.rows, A.cols, "a", pl, conj_t=trans_a)
    eb = ozaki.encode(B, B.rows, B.cols, "b", pl)
    res = ozaki.ResidueBuffer(m, n, pl.nmod, A.hi.re_buf.device)
    out = DDPlanar.empty(m, n, device=A.hi.re_buf.device)
    ozaki.gemm_residues(ea, eb, pl, res)
    ozaki.decode(res, ea, eb, pl, out)
    _counters["hp_calls"] += 1
    return out.to_ddmatrix() if host else out


def matmul_dd_fma(a, b, trans_a=False, out=None):
    """C = op(A) B in double-double on the FP64 pipe with FMA error-free
    transformations (csrc/ddgemm_fma.cu): the measured comparison point for
    the dd products (north_star item 2) — dd mode runs the
    Ozaki-II products, which measure faster.  a, b: DDPlanar."""
    from .matrix import DDPlanar
    m, k = (a.cols, a.rows) if trans_a else (a.rows, a.cols)
    if b.rows != k:
        raise ValueError("inner dimensions disagree: %d vs %d" % (k, b.rows))
    n = b.cols
    if out is None:
        out = DDPlanar.empty(m, n, device=a.hi.re_buf.device)
    _lib.call("sr_zgemm_dd_fma", _lib.SR_OP_C if trans_a else _lib.SR_OP_N, m, n, k, a.hi.re_ptr(), a.lo.re_ptr(),
              a.hi.im_ptr(), a.lo.im_ptr(), a.ld, b.hi.re_ptr(), b.lo.re_ptr(), b.hi.im_ptr(), b.lo.im_ptr(), b.ld,
              out.hi.re_ptr(), out.lo.re_ptr(), out.hi.im_ptr(), out.lo.im_ptr(), out.ld, _stream())
    _counters["hp_calls"] += 1
    return out


def matmul_hp(a, b, trans_a=False, alpha=1.0, diag_shift=0.0, out=None, trans_b=False):
    """C = alpha * op(A) B (+ diag_shift * I), FP64 complex planar.

    op(A) = A^H when trans_a (the reference materialises conj_t first,
    matmul.py:64; here the kernel reads A transposed from global memory).
    b may be real (no imaginary plane).  Double-double operands (DDMatrix,
    DDPlanar, anything with `.cells()`): the reference's dd product
    op(A) op(B) with trans_a / trans_b (matmul.py:52-81), see _matmul_dd."""
    if not isinstance(a, ZPlanar) and hasattr(a, "cells") or not isinstance(b, ZPlanar) and hasattr(b, "cells"):
        if alpha != 1.0 or diag_shift != 0.0 or out is not None:
            raise ValueError("dd products take no alpha / diag_shift / out")
        return _matmul_dd(a, b, trans_a, trans_b)
    if trans_b:
        raise NotImplementedError("trans_b is the dd-operand form")
    if a.is_real:
        raise ValueError("matmul_hp: A must be complex (a real A^H A is not on the path)")
    m = a.cols if trans_a else a.rows
    k = a.rows if trans_a else a.cols
    if b.rows != k:
        raise ValueError("inner dimensions disagree: %d vs %d" % (k, b.rows))
    n = b.cols
    if out is None:
        out = ZPlanar.empty(m, n, device=a.re_buf.device)
    _lib.call("sr_zgemm_f64", _lib.SR_OP_C if trans_a else _lib.SR_OP_N, m, n, k, float(alpha),
              float(diag_shift), a.re_ptr(), a.im_ptr(), a.ld, b.re_ptr(), b.im_ptr(), b.ld,
              out.re_ptr(), out.im_ptr(), out.ld, _stream())
    _counters["hp_calls"] += 1
    return out


def matmul_lp(a, b, m=None, n=None, k=None, out=None):
    """C = A B in complex64 (interleaved (rows, ld) tensors)."""
    m = a.shape[0] if m is None else m
    k = b.shape[0] if k is None else k
    n = b.shape[1] if n is None else n
    if out is None:
        out = lp_empty(m, n, device=a.device)
    _lib.call("sr_cgemm_c64", _lib.SR_OP_N, m, n, k, a.data_ptr(), a.shape[1], b.data_ptr(), b.shape[1],
              out.data_ptr(), out.shape[1], _stream())
    _counters["lp_calls"] += 1
    return out


_POWER_WS = {}


def spectral_norm_estimate(q_lp, n, rel_tol=1e-6, max_iters=200, group=8):
    """Largest singular value by power iteration on M^H M (matmul.py:117-142):
    the reference's fixed start vector 1 + (j mod 7)/8, stop when successive
    estimates agree to rel_tol or after max_iters.  M is the (n, ld) complex64
    lp matrix; the iteration runs in libsr (csrc/guards.cu, FP64 vectors) with
    the convergence test on the device — the host reads one small state
    record per group of `group` steps (one read for a near-unitary Q^)."""
    dev = q_lp.device
    key = (n, str(dev))
    ws = _POWER_WS.get(key)
    if ws is None:
        _POWER_WS.clear()
        ws = _POWER_WS[key] = torch.empty(_lib.load().sr_power_norm_workspace_bytes(n), dtype=torch.uint8,
                                          device=dev)
    state = ws[:40].view(torch.float64)
    done, first = 0, 1
    while done < max_iters:
        steps = min(group, max_iters - done)
        _lib.call("sr_power_norm_c64", n, q_lp.data_ptr(), q_lp.shape[1], first, steps, float(rel_tol),
                  ws.data_ptr(), ws.numel(), _stream())
        first = 0
        done += steps
        est, _prev, _nw, stop, _its = state.tolist()
        if stop:
            break
    return est
