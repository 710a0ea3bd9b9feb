"""Device time of each phase of one config-3 refinement (CUDA events recorded
at refine.py's phase marks): python tools/phase_times.py [n] [reps]."""
import collections
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2203_10879_b200 import RefineConfig, inputs, refine, refine_template  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
a, q = inputs.config_inputs(3, n=n)
ad = torch.from_numpy(np.ascontiguousarray(a)).cuda()
qd = torch.from_numpy(np.ascontiguousarray(q)).cuda()
cfg = RefineConfig(precision="fp64", tol_factor=10.0 / n, max_iters=10)
for _ in range(2):
    refine_template(ad, qd, cfg)
for r in range(reps):
    torch.cuda.synchronize()
    refine.PHASES = []
    refine_template(ad, qd, cfg)
    torch.cuda.synchronize()
    ph, refine.PHASES = refine.PHASES, None
    tot = collections.OrderedDict()
    seq = []
    for (l0, e0), (l1, e1) in zip(ph[:-1], ph[1:]):
        ms = e0.elapsed_time(e1)
        tot[l1] = tot.get(l1, 0.0) + ms
        seq.append("%s %.2f" % (l1, ms))
    print("total %.2f ms: " % ph[0][1].elapsed_time(ph[-1][1]) + ", ".join("%s %.2f" % kv for kv in tot.items()))
    if r == reps - 1:
        print("sequence: " + " | ".join(seq))
