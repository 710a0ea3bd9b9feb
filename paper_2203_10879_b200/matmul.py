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


def matmul_hp(a, b, trans_a=False, alpha=1.0, diag_shift=0.0, out=None):
    """C = alpha * op(A) B (+ diag_shift * I), FP64 complex planar.

    op(A) = A^H when trans_a (the reference materialises conj_t first,
    matmul.py:64; here the kernel reads A transposed from global memory).
    b may be real (no imaginary plane)."""
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


def spectral_norm_estimate(q_lp, n, rel_tol=1e-6, max_iters=200):
    """Largest singular value by power iteration on M^H M in lp (complex64),
    fixed start vector 1 + (j mod 7)/8 (matmul.py:117-142).  The two
    matrix-vector products per step are plain cuBLAS GEMVs (HBM-bound, 2 x 0.5
    GB at n = 8192): a guard on the entry, not a hot-path product."""
    dev = q_lp.device
    m = q_lp[:, :n]
    j = torch.arange(n, device=dev, dtype=torch.float32)
    v = (1.0 + torch.remainder(j, 7.0) / 8.0).to(torch.complex64)
    v = v / torch.linalg.vector_norm(v)
    prev = 0.0
    est = 0.0
    for _ in range(max_iters):
        u = torch.mv(m, v)
        w = torch.mv(m.mH, u)
        norms = torch.stack([torch.linalg.vector_norm(u), torch.linalg.vector_norm(w)]).double().cpu()
        est, nw = float(norms[0]), float(norms[1])
        if est == 0.0:
            return 0.0
        if nw == 0.0:
            return est
        v = w / nw
        if abs(est - prev) <= rel_tol * est:
            break
        prev = est
    return est
