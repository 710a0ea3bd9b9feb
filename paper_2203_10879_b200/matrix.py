"""Device containers for the two precisions of FP64 mode.

hp (complex128 in FP64 mode) matrices are stored PLANAR — separate float64
re / im planes — row-major with an even leading dimension, so the DMMA
GEMM can stage either plane with 16-byte cp.async granules and a real
matrix (config 3's A) is simply a matrix with no imaginary plane.  This is
the B200 counterpart of the reference's DDMatrix (four column-major float64
cell planes, /root/reference/pkg/src/ddschur/ddmatrix.py:29-66).

lp matrices (complex64) are interleaved torch complex64 tensors of shape
(n, ld) — the solver and the lp GEMM read (re, im) pairs as one float2.
"""
import numpy as np
import torch


def even(n):
    return n + (n & 1)


class ZPlanar:
    """Planar FP64 complex (or real, im is None) matrix on a CUDA device."""

    __slots__ = ("rows", "cols", "ld", "re_buf", "im_buf")

    def __init__(self, re_buf, im_buf, rows, cols):
        self.re_buf = re_buf
        self.im_buf = im_buf
        self.rows = rows
        self.cols = cols
        self.ld = re_buf.shape[1]

    @classmethod
    def empty(cls, rows, cols=None, device="cuda", real=False):
        cols = rows if cols is None else cols
        ld = even(max(cols, 1))
        re = torch.empty((rows, ld), dtype=torch.float64, device=device)
        im = None if real else torch.empty((rows, ld), dtype=torch.float64, device=device)
        return cls(re, im, rows, cols)

    @classmethod
    def from_any(cls, x, device="cuda", force_complex=False):
        """Copy a numpy / torch, real or complex 2-d matrix into planar form
        (exact embedding, like DDMatrix.from_lp, ddmatrix.py:75-82)."""
        if isinstance(x, ZPlanar):
            return x
        if isinstance(x, np.ndarray):
            x = torch.from_numpy(np.ascontiguousarray(x))
        if x.dim() != 2:
            raise ValueError("expected a 2-d array")
        rows, cols = x.shape
        real = not (x.is_complex() or force_complex)
        m = cls.empty(rows, cols, device=device, real=real)
        return cls.fill_from(m, x)

    @staticmethod
    def fill_from(m, x):
        """Copy a (rows, cols) torch matrix into the planes of m (on the current stream)."""
        device = m.re_buf.device
        cols = x.shape[1]
        if x.is_complex():
            xd = x.to(device=device, dtype=torch.complex128, non_blocking=True)
            m.re_buf[:, :cols].copy_(xd.real)
            m.im_buf[:, :cols].copy_(xd.imag)
        elif x.dtype == torch.float64:
            m.re_buf[:, :cols].copy_(x, non_blocking=True)
            if m.im_buf is not None:
                m.im_buf.zero_()
        else:
            m.re_buf[:, :cols].copy_(x.to(device=device, dtype=torch.float64, non_blocking=True))
            if m.im_buf is not None:
                m.im_buf.zero_()
        if m.ld != cols:
            m.re_buf[:, cols:].zero_()
            if m.im_buf is not None:
                m.im_buf[:, cols:].zero_()
        return m

    @property
    def shape(self):
        return (self.rows, self.cols)

    @property
    def is_real(self):
        return self.im_buf is None

    @property
    def re(self):
        return self.re_buf[:, : self.cols]

    @property
    def im(self):
        return None if self.im_buf is None else self.im_buf[:, : self.cols]

    def re_ptr(self):
        return self.re_buf.data_ptr()

    def im_ptr(self):
        return None if self.im_buf is None else self.im_buf.data_ptr()

    def to_complex(self, out=None):
        """complex128 (rows, cols) torch tensor on the same device (into out when given)."""
        im = self.im if self.im is not None else torch.zeros_like(self.re)
        if out is not None:
            return torch.complex(self.re, im, out=out)
        return torch.complex(self.re.contiguous(), im.contiguous())

    def to_numpy(self):
        return self.to_complex().cpu().numpy()

    def copy_(self, other):
        self.re_buf.copy_(other.re_buf)
        if self.im_buf is not None:
            self.im_buf.copy_(other.im_buf)
        return self


def lp_empty(rows, cols=None, device="cuda", dtype=torch.complex64):
    """Interleaved lp matrix (rows, ld) with an even leading dimension."""
    cols = rows if cols is None else cols
    return torch.empty((rows, even(max(cols, 1))), dtype=dtype, device=device)


class DDPlanar:
    """Double-double complex matrix on a CUDA device: two planar FP64 pairs,
    hi = (re_hi, im_hi) and lo = (re_lo, im_lo), each entry a normalised pair
    (|lo| <= ulp(hi) / 2).  The device counterpart of the reference's DDMatrix
    (/root/reference/pkg/src/ddschur/ddmatrix.py:29-66): same four planes,
    row-major instead of column-major."""

    __slots__ = ("hi", "lo")

    def __init__(self, hi, lo):
        self.hi = hi
        self.lo = lo

    @classmethod
    def empty(cls, rows, cols=None, device="cuda"):
        return cls(ZPlanar.empty(rows, cols, device=device), ZPlanar.empty(rows, cols, device=device))

    @classmethod
    def from_any(cls, x, device="cuda"):
        """Exact embedding (lo = 0) of a complex / real matrix, or a copy of
        a 4-plane (re_hi, re_lo, im_hi, im_lo) tuple (DDMatrix.cells order)."""
        if isinstance(x, DDPlanar):
            return x
        if hasattr(x, "cells") and not isinstance(x, ZPlanar):
            # the reference's DDMatrix (or ours): column-major cells, copied as row-major planes
            x = tuple(x.cells())
        if isinstance(x, (tuple, list)) and len(x) == 4:
            rh, rl, ih, il = (np.ascontiguousarray(c, dtype=np.float64) for c in x)
            return cls(ZPlanar.from_any(rh + 1j * ih, device=device, force_complex=True),
                       ZPlanar.from_any(rl + 1j * il, device=device, force_complex=True))
        hi = ZPlanar.from_any(x, device=device, force_complex=True)
        lo = ZPlanar.empty(hi.rows, hi.cols, device=device)
        lo.re_buf.zero_()
        lo.im_buf.zero_()
        return cls(hi, lo)

    @property
    def rows(self):
        return self.hi.rows

    @property
    def cols(self):
        return self.hi.cols

    @property
    def shape(self):
        return self.hi.shape

    @property
    def ld(self):
        return self.hi.ld

    def cells(self):
        """(re_hi, re_lo, im_hi, im_lo) device views, DDMatrix.cells order."""
        return self.hi.re, self.lo.re, self.hi.im, self.lo.im

    def to_numpy_cells(self):
        return tuple(c.cpu().numpy() for c in self.cells())


class ColView:
    """Columns j0..j1 of a ZPlanar, as a strided view with the parent's
    leading dimension (the column block a rank owns in the sharded driver)."""

    __slots__ = ("parent", "j0", "j1")

    def __init__(self, parent, j0, j1):
        self.parent, self.j0, self.j1 = parent, j0, j1

    @property
    def rows(self):
        return self.parent.rows

    @property
    def cols(self):
        return self.j1 - self.j0

    @property
    def ld(self):
        return self.parent.ld

    @property
    def is_real(self):
        return self.parent.is_real

    @property
    def re_buf(self):
        return self.parent.re_buf

    def re_ptr(self):
        return self.parent.re_ptr() + 8 * self.j0

    def im_ptr(self):
        p = self.parent.im_ptr()
        return None if p is None else p + 8 * self.j0
