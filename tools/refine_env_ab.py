"""Interleaved A/B of a whole config-3 refinement under two settings of one
environment variable that libsr reads at every launch (e.g. SR_OZ_WIDE).
Usage: python tools/refine_env_ab.py VAR VALUE_A VALUE_B [n] [reps]"""
import os
import statistics
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2203_10879_b200 import RefineConfig, inputs, refine_template  # noqa: E402

var, va, vb = sys.argv[1:4]
n = int(sys.argv[4]) if len(sys.argv) > 4 else 8192
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 5
a, q = inputs.config_inputs(3, n=n)
ad = torch.from_numpy(np.ascontiguousarray(a)).cuda()
qd = torch.from_numpy(np.ascontiguousarray(q)).cuda()
cfg = RefineConfig(precision="fp64", tol_factor=10.0 / n, max_iters=10)
t = {va: [], vb: []}
for r in range(reps + 1):
    for v in (va, vb):
        os.environ[var] = v
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        pair, rep = refine_template(ad, qd, cfg)
        torch.cuda.synchronize()
        if r:
            t[v].append(time.perf_counter() - t0)
for v in (va, vb):
    print("%s=%s: median %.4f s  min %.4f s  (%s)" % (var, v, statistics.median(t[v]), min(t[v]),
                                                       ", ".join("%.4f" % x for x in t[v])), flush=True)
