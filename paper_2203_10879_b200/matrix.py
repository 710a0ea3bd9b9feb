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
        if x.is_complex():
            xd = x.to(device=device, dtype=torch.complex128, non_blocking=True)
            m.re_buf[:, :cols].copy_(xd.real)
            m.im_buf[:, :cols].copy_(xd.imag)
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

    def to_complex(self):
        """complex128 (rows, cols) torch tensor on the same device."""
        im = self.im if self.im is not None else torch.zeros_like(self.re)
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
