"""Config-3 refinement with Q encoded at a lower beta (ozaki.HP_BETA_Q): moduli,
time, iterations and final residuals.  Usage: python tools/beta_probe.py [n] [beta_q ...]"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2203_10879_b200 import RefineConfig, inputs, ozaki, refine_template  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
betas = [int(b) for b in sys.argv[2:]] or [58, 57]
a, q = inputs.config_inputs(3, n=n)
ad = torch.from_numpy(np.ascontiguousarray(a)).cuda()
qd = torch.from_numpy(np.ascontiguousarray(q)).cuda()
cfg = RefineConfig(precision="fp64", tol_factor=10.0 / n, max_iters=10)
for bq in betas:
    ozaki.HP_BETA_Q = bq
    from paper_2203_10879_b200 import refine as R
    R._WS_CACHE.clear()
    times = []
    for rep in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        pair, rep_ = refine_template(ad, qd, cfg)
        torch.cuda.synchronize()
        times.append(time.perf_counter() - t0)
    R.PHASES = []
    refine_template(ad, qd, cfg)
    torch.cuda.synchronize()
    ph, R.PHASES = R.PHASES, None
    acc = {}
    for (l0, e0), (l1, e1) in zip(ph, ph[1:]):
        acc[l1] = acc.get(l1, 0.0) + e0.elapsed_time(e1)
    print("  phases: " + ", ".join("%s %.1f ms" % kv for kv in acc.items()), flush=True)
    print("beta_q %d: nmod(QhQ) %d, time %.4f s (min of 3 after warm-up), iterations %d, history %s" % (
        bq, ozaki.plan(n, bq, bq, True).nmod, min(times[1:]), rep_.iterations,
        ["%.3e / %.3e" % (h[0] / np.linalg.norm(a), h[1]) for h in rep_.residual_history]), flush=True)
