"""Time-to-refine of BASELINE configs 1 and 2 (FP64 mode, inputs resident on the device)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2203_10879_b200 import RefineConfig, inputs, refine_template  # noqa: E402

for cfgno in (1, 2):
    a, q = inputs.config_inputs(cfgno)
    n = a.shape[0]
    ad, qd = torch.from_numpy(np.ascontiguousarray(a)).cuda(), torch.from_numpy(np.ascontiguousarray(q)).cuda()
    cfg = RefineConfig(precision="fp64", tol_factor=10.0 / n, max_iters=10)
    ts = []
    for _ in range(5):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        pair, rep = refine_template(ad, qd, cfg)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    print("config %d (n=%d): %.4f s (min of 4 after warm-up), %s, %d iterations, final relE %.2e" % (
        cfgno, n, min(ts[1:]), rep.status.value, rep.iterations,
        rep.residual_history[-1][0] / np.linalg.norm(a)), flush=True)
