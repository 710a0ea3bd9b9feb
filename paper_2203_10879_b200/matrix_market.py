"""Matrix Market exchange format, the reference's disk
format (/root/reference/pkg/src/ddschur/mmio.py:137-217).

Reading accepts coordinate and array files, real / complex / integer fields,
general / symmetric storage, densified into double-double planes (hi, lo)
with exact decimal parsing: each value is the nearest double-double of the
decimal text, so files written at 36 significant digits round-trip bit for
bit.  Writing emits the dense array format, general symmetry, column-major
order: 36 significant digits per component for double-double input, 17 for
binary64.  Host-side (numpy) I/O; DDPlanar / torch inputs are read back to
the host first.
"""
from decimal import Decimal, localcontext
from fractions import Fraction

import numpy as np

_FORMATS = ("coordinate", "array")
_FIELDS = ("real", "complex", "integer")
_SYMMETRIES = ("general", "symmetric")


class MatrixMarketError(ValueError):
    """Malformed Matrix Market content: header, sizes, indices or values."""


def _header(line):
    parts = line.split()
    if len(parts) != 5 or parts[0].lower() != "%%matrixmarket":
        raise MatrixMarketError("not a Matrix Market header: %r" % line.strip())
    obj, fmt, field, sym = (p.lower() for p in parts[1:])
    if obj != "matrix":
        raise MatrixMarketError("unsupported object %r" % obj)
    if fmt not in _FORMATS:
        raise MatrixMarketError("unsupported format %r" % fmt)
    if field not in _FIELDS:
        raise MatrixMarketError("unsupported field %r" % field)
    if sym not in _SYMMETRIES:
        raise MatrixMarketError("unsupported symmetry %r" % sym)
    return fmt, field, sym


def _dd(tok):
    """Nearest double-double (hi, lo) of a decimal token (exact rational arithmetic)."""
    try:
        f = Fraction(tok)
    except (ValueError, ZeroDivisionError):
        raise MatrixMarketError("bad numeric value %r" % tok)
    hi = float(f)
    lo = float(f - Fraction(hi))
    s = hi + lo  # normalise (two-sum)
    bb = s - hi
    return s, (hi - (s - bb)) + (lo - bb)


def _index(tok):
    try:
        return int(tok)
    except ValueError:
        raise MatrixMarketError("bad index %r" % tok)


def _values(toks, field):
    want = 2 if field == "complex" else 1
    if len(toks) != want:
        raise MatrixMarketError("expected %d value(s), got %r" % (want, toks))
    re = _dd(toks[0])
    im = _dd(toks[1]) if field == "complex" else (0.0, 0.0)
    return re, im


def _data_lines(path):
    with open(path, "r", encoding="ascii") as f:
        raw = f.readlines()
    if not raw:
        raise MatrixMarketError("empty file")
    fmt, field, sym = _header(raw[0])
    data = [ln for ln in raw[1:] if ln.strip() and not ln.lstrip().startswith("%")]
    if not data:
        raise MatrixMarketError("missing size line")
    return fmt, field, sym, data


def read_matrix_market(path):
    """-> (re_hi, re_lo, im_hi, im_lo) float64 planes (the DDMatrix.cells()
    order, accepted by refine_template in dd mode)."""
    fmt, field, sym, data = _data_lines(path)
    size = [_index(t) for t in data[0].split()]
    if len(size) != (3 if fmt == "coordinate" else 2):
        raise MatrixMarketError("malformed size line %r" % data[0])
    if min(size[:2]) < 1 or (fmt == "coordinate" and size[2] < 0):
        raise MatrixMarketError("bad sizes %r" % (size,))
    rows, cols = size[0], size[1]
    if sym == "symmetric" and rows != cols:
        raise MatrixMarketError("symmetric storage needs a square matrix")
    planes = [np.zeros((rows, cols)) for _ in range(4)]

    def put(i, j, re, im):
        planes[0][i, j], planes[1][i, j] = re
        planes[2][i, j], planes[3][i, j] = im

    body = data[1:]
    if fmt == "coordinate":
        nnz = size[2]
        if len(body) != nnz:
            raise MatrixMarketError("expected %d entries, found %d" % (nnz, len(body)))
        seen = set()
        for ln in body:
            toks = ln.split()
            if len(toks) < 3:
                raise MatrixMarketError("malformed entry %r" % ln)
            i, j = _index(toks[0]) - 1, _index(toks[1]) - 1
            if not (0 <= i < rows and 0 <= j < cols):
                raise MatrixMarketError("index out of range in %r" % ln)
            if sym == "symmetric" and j > i:
                raise MatrixMarketError("symmetric storage lists the lower triangle only: %r" % ln)
            if (i, j) in seen:
                raise MatrixMarketError("duplicate entry (%d, %d)" % (i + 1, j + 1))
            seen.add((i, j))
            re, im = _values(toks[2:], field)
            put(i, j, re, im)
            if sym == "symmetric" and i != j:
                put(j, i, re, im)
    else:
        cells = [(i, j) for j in range(cols) for i in range(rows) if sym == "general" or i >= j]
        if len(body) != len(cells):
            raise MatrixMarketError("expected %d values, found %d" % (len(cells), len(body)))
        for (i, j), ln in zip(cells, body):
            re, im = _values(ln.split(), field)
            put(i, j, re, im)
            if sym == "symmetric" and i != j:
                put(j, i, re, im)
    return tuple(planes)


def header_metadata(path):
    """(format, field, symmetry, sizes) without densifying; sizes (rows, cols,
    nnz) for coordinate files, (rows, cols) for array files."""
    fmt, field, sym, data = _data_lines(path)
    toks = data[0].split()
    if len(toks) != (3 if fmt == "coordinate" else 2):
        raise MatrixMarketError("malformed size line %r" % data[0])
    return fmt, field, sym, tuple(_index(t) for t in toks)


def _dd_string(hi, lo, digits=36):
    with localcontext() as ctx:
        ctx.prec = digits
        return str(Decimal(hi) + Decimal(lo))


def write_matrix_market(path, m, comment=None):
    """Dense array-format, general-symmetry file.  m: a 4-plane dd tuple
    (re_hi, re_lo, im_hi, im_lo) or a DDPlanar (36 digits per component), or
    any 2-d numpy / torch array (binary64, 17 digits).  The field is complex
    when any imaginary part is nonzero."""
    from .matrix import DDPlanar
    if isinstance(m, DDPlanar):
        m = m.to_numpy_cells()
    if isinstance(m, tuple) and len(m) == 4:
        rh, rl, ih, il = (np.asarray(x, dtype=np.float64) for x in m)
        rows, cols = rh.shape
        cplx = bool(np.any(ih != 0.0) or np.any(il != 0.0))

        def render(i, j):
            s = _dd_string(rh[i, j], rl[i, j])
            return "%s %s" % (s, _dd_string(ih[i, j], il[i, j])) if cplx else s
    else:
        if hasattr(m, "detach"):
            m = m.detach().cpu().numpy()
        arr = np.asarray(m)
        if arr.ndim != 2:
            raise MatrixMarketError("need a 2-d matrix")
        rows, cols = arr.shape
        cplx = bool(np.iscomplexobj(arr) and np.any(arr.imag != 0.0))

        def render(i, j):
            v = complex(arr[i, j])
            return "%.16e %.16e" % (v.real, v.imag) if cplx else "%.16e" % v.real
    lines = ["%%%%MatrixMarket matrix array %s general" % ("complex" if cplx else "real")]
    if comment:
        lines += ["%% %s" % c for c in str(comment).splitlines()]
    lines.append("%d %d" % (rows, cols))
    lines += [render(i, j) for j in range(cols) for i in range(rows)]
    with open(path, "w", encoding="ascii") as f:
        f.write("\n".join(lines) + "\n")


__all__ = ["MatrixMarketError", "read_matrix_market", "header_metadata", "write_matrix_market"]
