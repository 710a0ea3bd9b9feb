"""The reference's matrix-core boundary (ddschur.ddmatrix) on the B200.

  DDMatrix            /root/reference/pkg/src/ddschur/ddmatrix.py:29-150
  precision_convert   ddmatrix.py:157-161
  stril_extract       ddmatrix.py:190-209
  frobenius_norm      ddmatrix.py:216-251

`DDMatrix` is the reference's HOST container — four column-major float64
planes (re_hi, re_lo, im_hi, im_lo) — so results can be handed to code
written against the reference (its verify_pair, its tests) and reference
DDMatrix objects (anything with `.cells()`) are accepted everywhere.  Its
arithmetic (+, -, scale) and the helpers below run on the GPU
(csrc/dd_ops.cu) and are BIT-IDENTICAL to the reference's numpy / numba
kernels for finite operands; the device twin is `DDPlanar` (row-major planes,
matrix.py), with `to_device()` / `DDPlanar.to_ddmatrix()` between the two.
"""
import numpy as np
import torch

from . import _lib
from .matrix import DDPlanar, ZPlanar


def _stream():
    return torch.cuda.current_stream().cuda_stream


def _fortran(a):
    return np.asfortranarray(a, dtype=np.float64)


class DDScalar:
    """A double-double real (hi, lo): frobenius_norm's result, the reference's
    DDReal (dd.py:187-…) reduced to what the boundary needs; float(x) = hi."""

    __slots__ = ("hi", "lo")

    def __init__(self, hi, lo=0.0):
        self.hi, self.lo = float(hi), float(lo)

    def __float__(self):
        return self.hi

    def __eq__(self, other):
        if isinstance(other, DDScalar):
            return self.hi == other.hi and self.lo == other.lo
        return self.hi == float(other) and self.lo == 0.0

    def __repr__(self):
        return "DDScalar(%r, %r)" % (self.hi, self.lo)


class DDMatrix:
    """Host double-double complex matrix, the reference's container
    (ddmatrix.py:29-150): four column-major float64 cells, normalised pairs."""

    __slots__ = ("re_hi", "re_lo", "im_hi", "im_lo")

    def __init__(self, re_hi, re_lo, im_hi, im_lo):
        self.re_hi = _fortran(re_hi)
        self.re_lo = _fortran(re_lo)
        self.im_hi = _fortran(im_hi)
        self.im_lo = _fortran(im_lo)
        shape = self.re_hi.shape
        if len(shape) != 2 or any(c.shape != shape for c in self.cells()):
            raise ValueError("cell arrays must share one 2-d shape")

    def cells(self):
        return self.re_hi, self.re_lo, self.im_hi, self.im_lo

    @property
    def rows(self):
        return self.re_hi.shape[0]

    @property
    def cols(self):
        return self.re_hi.shape[1]

    @property
    def shape(self):
        return self.re_hi.shape

    @classmethod
    def zeros(cls, rows, cols=None):
        cols = rows if cols is None else cols
        return cls(*(np.zeros((rows, cols), order="F") for _ in range(4)))

    @classmethod
    def eye(cls, n, scale=1.0):
        m = cls.zeros(n, n)
        np.fill_diagonal(m.re_hi, float(scale))
        return m

    @classmethod
    def from_lp(cls, a):
        """Exact embedding of a complex128 (or real) matrix; lo cells are 0."""
        a = np.asarray(a)
        if a.ndim != 2:
            raise ValueError("expected a 2-d array")
        z = np.zeros(a.shape, order="F")
        return cls(a.real, z.copy(), a.imag if np.iscomplexobj(a) else z.copy(), z.copy())

    @classmethod
    def from_cells(cls, x):
        """Any object with the reference's `.cells()` (e.g. ddschur.DDMatrix)."""
        return cls(*x.cells())

    def to_lp(self):
        return np.asfortranarray(self.re_hi + 1j * self.im_hi)

    def copy(self):
        return DDMatrix(*(c.copy(order="F") for c in self.cells()))

    def conj_t(self):
        return DDMatrix(self.re_hi.T, self.re_lo.T, -self.im_hi.T, -self.im_lo.T)

    def is_finite(self):
        return all(np.isfinite(c).all() for c in self.cells())

    def bits_equal(self, other):
        return all(np.array_equal(x, y, equal_nan=True) for x, y in zip(self.cells(), other.cells()))

    def to_device(self, device="cuda"):
        return DDPlanar.from_any(self.cells(), device=device)

    # ---- arithmetic on the GPU, bit-identical to the reference's v_add / v_sub / v_mul_d
    def __add__(self, other):
        if not _is_dd(other):
            return NotImplemented
        return dd_add(self, other).to_ddmatrix()

    def __sub__(self, other):
        if not _is_dd(other):
            return NotImplemented
        return dd_add(self, other, negate=True).to_ddmatrix()

    def __neg__(self):
        return DDMatrix(-self.re_hi, -self.re_lo, -self.im_hi, -self.im_lo)

    def scale(self, s):
        if isinstance(s, DDScalar):
            if s.lo != 0.0:
                raise NotImplementedError("scaling by a double-double scalar")
            s = s.hi
        return dd_scale(self, float(s)).to_ddmatrix()

    def __repr__(self):
        return "DDMatrix(%d x %d)" % self.shape


def _is_dd(x):
    return isinstance(x, (DDMatrix, DDPlanar)) or (hasattr(x, "cells") and not isinstance(x, ZPlanar))


def as_ddplanar(x, device="cuda"):
    """DDPlanar view/copy of a dd matrix (DDPlanar, DDMatrix, anything with
    `.cells()`, a 4-plane tuple) or exact embedding of an lp matrix."""
    if isinstance(x, DDPlanar):
        return x
    if hasattr(x, "cells") and not isinstance(x, ZPlanar):
        return DDPlanar.from_any(tuple(x.cells()), device=device)
    return DDPlanar.from_any(x, device=device)


def _to_ddmatrix(self, cls=None):
    """Host DDMatrix (column-major cells) of a device dd matrix; cls: another
    container with the reference's constructor, e.g. ddschur.DDMatrix."""
    cells = [np.asfortranarray(c.cpu().numpy()) for c in self.cells()]
    return (cls or DDMatrix)(*cells)


DDPlanar.to_ddmatrix = _to_ddmatrix
DDPlanar.to_lp = lambda self: self.hi  # binary64 rounding of normalised pairs: the hi planes


def dd_add(x, y, negate=False):
    """x + y (x - y with negate) in dd on the device -> DDPlanar."""
    X = as_ddplanar(x)
    Y = as_ddplanar(y, device=X.hi.re_buf.device)
    if X.shape != Y.shape:
        raise ValueError("shape mismatch %s vs %s" % (X.shape, Y.shape))
    m, n = X.shape
    Z = DDPlanar.empty(m, n, device=X.hi.re_buf.device)
    st = _stream()
    for part in ("re", "im"):
        xh, xl = getattr(X.hi, part + "_buf"), getattr(X.lo, part + "_buf")
        yh, yl = getattr(Y.hi, part + "_buf"), getattr(Y.lo, part + "_buf")
        zh, zl = getattr(Z.hi, part + "_buf"), getattr(Z.lo, part + "_buf")
        _lib.call("sr_dd_add", m, n, xh.data_ptr(), xl.data_ptr(), X.ld, yh.data_ptr(), yl.data_ptr(), Y.ld,
                  1 if negate else 0, zh.data_ptr(), zl.data_ptr(), Z.ld, st)
    return Z


def dd_scale(x, s):
    """s * x in dd (s a binary64 scalar) on the device -> DDPlanar."""
    X = as_ddplanar(x)
    m, n = X.shape
    Z = DDPlanar.empty(m, n, device=X.hi.re_buf.device)
    st = _stream()
    for part in ("re", "im"):
        xh, xl = getattr(X.hi, part + "_buf"), getattr(X.lo, part + "_buf")
        zh, zl = getattr(Z.hi, part + "_buf"), getattr(Z.lo, part + "_buf")
        _lib.call("sr_dd_scale", m, n, xh.data_ptr(), xl.data_ptr(), X.ld, float(s), zh.data_ptr(),
                  zl.data_ptr(), Z.ld, st)
    return Z


def precision_convert(m):
    """lp matrix -> DDMatrix (exact) or DDMatrix -> lp matrix (rounded = hi)."""
    if isinstance(m, DDMatrix):
        return m.to_lp()
    if isinstance(m, DDPlanar):
        return m.hi.to_complex()
    if hasattr(m, "cells"):
        return DDMatrix.from_cells(m).to_lp()
    return DDMatrix.from_lp(m)


def _split_plane(src, ld_src, e, t, m, n, st):
    _lib.call("sr_stril_split_f64", m, n, src.data_ptr(), ld_src, e.data_ptr(), e.shape[1], t.data_ptr(),
              t.shape[1], st)


def stril_extract(m):
    """(E, T): E the strictly lower part, T the rest, bit for bit (pure
    masking, E + T == m).  Returns the kind it was given: DDMatrix /
    DDPlanar pairs, numpy (column-major, like the reference) or torch."""
    st = _stream()
    if _is_dd(m):
        host = not isinstance(m, DDPlanar)
        X = as_ddplanar(m)
        rows, cols = X.shape
        if rows != cols:
            raise ValueError("stril_extract needs a square matrix")
        dev = X.hi.re_buf.device
        E, T = DDPlanar.empty(rows, cols, device=dev), DDPlanar.empty(rows, cols, device=dev)
        for src, e, t in ((X.hi.re_buf, E.hi.re_buf, T.hi.re_buf), (X.hi.im_buf, E.hi.im_buf, T.hi.im_buf),
                          (X.lo.re_buf, E.lo.re_buf, T.lo.re_buf), (X.lo.im_buf, E.lo.im_buf, T.lo.im_buf)):
            _split_plane(src, X.ld, e, t, rows, cols, st)
        return (E.to_ddmatrix(), T.to_ddmatrix()) if host else (E, T)
    is_np = not torch.is_tensor(m)
    x = torch.from_numpy(np.ascontiguousarray(m)) if is_np else m
    if x.dim() != 2 or x.shape[0] != x.shape[1]:
        raise ValueError("stril_extract needs a square matrix")
    dev = x.device if x.is_cuda else torch.device("cuda")
    xd = x.to(dev)
    planes = [torch.view_as_real(xd)[..., k].contiguous() for k in (0, 1)] if xd.is_complex() else \
        [xd.to(torch.float64).contiguous()]
    outs_e, outs_t = [], []
    for p in planes:
        e, t = torch.empty_like(p), torch.empty_like(p)
        _split_plane(p, p.shape[1], e, t, p.shape[0], p.shape[1], st)
        outs_e.append(e)
        outs_t.append(t)
    if xd.is_complex():
        e, t = torch.complex(*outs_e).to(x.dtype), torch.complex(*outs_t).to(x.dtype)
    else:
        e, t = outs_e[0].to(x.dtype), outs_t[0].to(x.dtype)
    if is_np:
        return np.asfortranarray(e.cpu().numpy()), np.asfortranarray(t.cpu().numpy())
    return (e, t) if x.is_cuda else (e.cpu(), t.cpu())


def frobenius_norm(m):
    """Frobenius norm accumulated in double-double over column-major order
    with the reference's fixed pairwise tree -> DDScalar (bit-identical to
    the reference's DDReal for finite inputs).  m: DDMatrix / DDPlanar /
    anything with `.cells()`, or an lp matrix (numpy, torch, ZPlanar)."""
    st = _stream()
    if _is_dd(m):
        X = as_ddplanar(m)
        rh, rl, ih, il = X.hi.re_buf, X.lo.re_buf, X.hi.im_buf, X.lo.im_buf
        rows, cols, ld, dev = X.rows, X.cols, X.ld, rh.device
        ptrs = (rh.data_ptr(), rl.data_ptr(), ih.data_ptr(), il.data_ptr())
    else:
        Z = m if isinstance(m, ZPlanar) else ZPlanar.from_any(m)
        rows, cols, ld, dev = Z.rows, Z.cols, Z.ld, Z.re_buf.device
        ptrs = (Z.re_ptr(), None, Z.im_ptr(), None)
    lib = _lib.load()
    ws = torch.empty(lib.sr_fro_norm_dd_workspace_bytes(rows * cols), dtype=torch.uint8, device=dev)
    out = torch.zeros(2, dtype=torch.float64, device=dev)
    _lib.call("sr_fro_norm_dd", rows, cols, *ptrs, ld, out.data_ptr(), ws.data_ptr(), ws.numel(), st)
    hi, lo = out.cpu().tolist()
    return DDScalar(hi, lo)


__all__ = ["DDMatrix", "DDScalar", "as_ddplanar", "dd_add", "dd_scale", "frobenius_norm", "precision_convert",
           "stril_extract"]
