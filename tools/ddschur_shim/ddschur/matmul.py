"""ddschur.matmul: dd products of DDMatrix operands on the int8 tensor cores."""
from paper_2203_10879_b200.matmul import counters, matmul_hp, matmul_lp, reset_counters  # noqa: F401
