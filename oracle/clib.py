"""ORACLE — test infrastructure only.

ctypes binding of `oracle/_build/liboracle.so` (built by `oracle/Makefile`
from `trisolve_oracle.c` and `ddgemm_oracle.c`, the plain-C restatements
of `trisolve.py:121-262` and `_numba_kernels.py:18-46`).
"""
import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle.so")
_lib = None


class SeparationError(Exception):
    """Mirror of ddschur.trisolve.SeparationError (trisolve.py:50-51)."""


class NonFiniteError(Exception):
    """Mirror of ddschur.trisolve.NonFiniteError (trisolve.py:54-55)."""


def build():
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        _lib = ctypes.CDLL(_LIB_PATH)
        p = ctypes.c_void_p
        for suf, real in (("c128", ctypes.c_double), ("c64", ctypes.c_float)):
            f = getattr(_lib, "oracle_solve_block_" + suf)
            f.argtypes = [ctypes.c_int, p, p, p, ctypes.c_int, real,
                          ctypes.POINTER(ctypes.c_longlong)]
            f.restype = ctypes.c_int
        _lib.oracle_gemm_dd.argtypes = [ctypes.c_int] * 4 + [p] * 12
        _lib.oracle_gemm_dd.restype = None
    return _lib


def solve_block(t, e, n_min=4, clip_threshold=None, dtype=np.complex128):
    """solve_block (trisolve.py:243-262) restated in C; returns (l, clipped).

    dtype selects the arithmetic: complex128 is the reference's binary64
    solver, complex64 the FP64-mode lp solver.
    """
    t = np.ascontiguousarray(t, dtype=dtype)
    e = np.ascontiguousarray(e, dtype=dtype)
    n = t.shape[0]
    if t.shape != (n, n) or e.shape != (n, n):
        raise ValueError("t and e must be square and of equal shape")
    l = np.zeros((n, n), dtype=dtype)
    clipped = ctypes.c_longlong(0)
    suf = "c128" if dtype == np.complex128 else "c64"
    f = getattr(lib(), "oracle_solve_block_" + suf)
    clip = 0.0 if clip_threshold is None else float(clip_threshold)
    rc = f(n, t.ctypes.data, e.ctypes.data, l.ctypes.data, int(n_min), clip,
           ctypes.byref(clipped))
    if rc == 1:
        raise ValueError("bad triangular problem (shape/structure/n_min)")
    if rc == 2:
        raise SeparationError("diagonal separation is exactly zero")
    if rc == 3:
        raise NonFiniteError("solution contains non-finite entries")
    return l, int(clipped.value)


def gemm_dd(a, b, panel=32):
    """Reference gemm_hp (numba kernel) restated in C; a, b are 4-tuples of
    (re_hi, re_lo, im_hi, im_lo) float64 planes; returns the 4 output planes."""
    a = [np.ascontiguousarray(x, dtype=np.float64) for x in a]
    b = [np.ascontiguousarray(x, dtype=np.float64) for x in b]
    m, k = a[0].shape
    k2, n = b[0].shape
    if k != k2:
        raise ValueError("inner dimensions disagree")
    out = [np.zeros((m, n)) for _ in range(4)]
    lib().oracle_gemm_dd(m, n, k, panel, *(x.ctypes.data for x in a),
                         *(x.ctypes.data for x in b), *(x.ctypes.data for x in out))
    return tuple(out)
