"""ORACLE — test / benchmark infrastructure only (the CPU baseline).

A BLAS-backed CPU port of the reference's low-precision solver
stril(T L - L T) = -E, used where the plain-C restatement
(oracle/trisolve_oracle.c, the parity checker) is too slow: the timed CPU
baseline of bench.py at n = 2048 … 8192.  Same algorithm, faster kernels:

  solve_block / _block_solve  /root/reference/pkg/src/ddschur/trisolve.py:223-262
      recursive halving at n1 = n // 2, identical split points;
  _stril_inplace_add          trisolve.py:217-220
      the two strict-lower updates E11 += stril(T12 X), E22 -= stril(X T12)
      as BLAS GEMMs (the reference calls matmul_lp, a parallel GEMM);
  _sylvester_tri              trisolve.py:164-196
      T22 X - X T11 = C for upper-triangular T22, T11: the reference solves it
      column by column (shifted back substitution); here by recursive
      splitting of the larger dimension (Jonsson–Kågström RECSY) down to
      LAPACK ?trsyl leaves (the same triangular Sylvester equation solved by
      the same substitution order inside a leaf), with the coupling terms as
      GEMMs.  The solution is the same matrix up to rounding;
  subproblems n <= leaf       the C restatement itself (Algorithm 2 leaves,
                              trisolve.py:121-145, and the same recursion).

No clipping (clip_threshold must be None: the benchmark workload never
clips) — the clip-semantics parity lives in the C restatement.
tests/test_oracle.py pins this port to the C restatement.
"""
import numpy as np
import scipy.linalg.lapack as lapack

from . import clib

SYLV_LEAF = 96    # ?trsyl leaf size (both dimensions)
BLOCK_LEAF = 128  # subproblems handed to the C restatement


def _trsyl(dtype):
    return lapack.ctrsyl if dtype == np.complex64 else lapack.ztrsyl


def sylvester_tri(t22, t11, c):
    """X with T22 X - X T11 = C (T22, T11 upper triangular), trisolve.py:164-196."""
    m, p = c.shape
    if m <= SYLV_LEAF and p <= SYLV_LEAF:
        x, scale, info = _trsyl(c.dtype)(t22, t11, c, trana="N", tranb="N", isgn=-1)
        if info < 0:
            raise ValueError("?trsyl argument %d" % -info)
        if info == 1:  # perturbed pivots: exactly equal eigenvalues (trisolve.py:185-189)
            raise clib.SeparationError("zero pivot in shifted triangular solve")
        return x if scale == 1.0 else x / scale
    if m >= p:
        m1 = m // 2
        x2 = sylvester_tri(t22[m1:, m1:], t11, c[m1:])
        x1 = sylvester_tri(t22[:m1, :m1], t11, c[:m1] - t22[:m1, m1:] @ x2)
        return np.vstack((x1, x2))
    p1 = p // 2
    x1 = sylvester_tri(t22, t11[:p1, :p1], c[:, :p1])
    x2 = sylvester_tri(t22, t11[p1:, p1:], c[:, p1:] + x1 @ t11[:p1, p1:])
    return np.hstack((x1, x2))


def _block(t, e, l, n_min):
    n = t.shape[0]
    if n <= BLOCK_LEAF:
        sub, _ = clib.solve_block(t, e, n_min=n_min, dtype=t.dtype)
        l[:, :] = sub
        return
    n1 = n // 2
    t11, t12, t22 = t[:n1, :n1], t[:n1, n1:], t[n1:, n1:]
    x = sylvester_tri(np.ascontiguousarray(t22), np.ascontiguousarray(t11), -e[n1:, :n1])
    l[n1:, :n1] = x
    e[:n1, :n1] += np.tril(t12 @ x, -1)
    e[n1:, n1:] -= np.tril(x @ t12, -1)
    _block(t11, e[:n1, :n1], l[:n1, :n1], n_min)
    _block(t22, e[n1:, n1:], l[n1:, n1:], n_min)


def solve_block(t, e, n_min=4, dtype=np.complex64):
    """solve_block (trisolve.py:243-262) -> L; raises clib.SeparationError /
    clib.NonFiniteError like the restatement."""
    t = np.ascontiguousarray(t, dtype=dtype)
    e = np.array(e, dtype=dtype, copy=True)
    n = t.shape[0]
    d = np.diagonal(t)
    if np.unique(d).size != n:
        raise clib.SeparationError("diagonal separation is exactly zero")
    l = np.zeros((n, n), dtype=dtype)
    with np.errstate(over="ignore", invalid="ignore"):
        _block(t, e, l, n_min)
    if not np.isfinite(l.view(l.real.dtype)).all():
        raise clib.NonFiniteError("solution contains non-finite entries")
    return l
