"""Residual history of one config-3-family refinement (FP64 mode) at size n:
python tools/history_probe.py [n]  (env switches of the solver apply)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2203_10879_b200 import RefineConfig, ZPlanar, inputs, refine_template  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
a = inputs.gaussian_real(n, 0)
q = inputs.cached_qhat("c3_n%d_s0" % n, a).astype(np.complex128)
A, Q = ZPlanar.from_any(a), ZPlanar.from_any(q)
cfg = RefineConfig(precision="fp64", tol_factor=10.0 / n, max_iters=10)
norm_a = float(np.linalg.norm(a))
for rep in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    pair, r = refine_template(A, Q, cfg)
    dt = time.perf_counter() - t0
print("n=%d %s it=%d skip=%s %.1f ms; relE history: %s; ortho: %s" % (
    n, r.status.value, r.iterations, r.skip_fired, dt * 1e3,
    " ".join("%.2e" % (e / norm_a) for e, _ in r.residual_history),
    " ".join("%.2e" % y for _, y in r.residual_history)), flush=True)
