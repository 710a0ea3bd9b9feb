"""ddschur.ddmatrix: the host container and the bit-identical GPU helpers."""
from paper_2203_10879_b200.ddmatrix import DDMatrix, frobenius_norm, precision_convert, stril_extract  # noqa: F401
