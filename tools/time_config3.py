"""Time whole config-3 refinements (device-resident inputs) in this process:
python tools/time_config3.py [reps] [n] -> one line 'median min' in seconds.
Used by tools/lib_ab.sh to A/B two builds of libsr (SR_LIB_PATH) on one box."""
import statistics
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2203_10879_b200 import RefineConfig, inputs, refine_template  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
n = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
a, q = inputs.config_inputs(3, n=n)
ad = torch.from_numpy(np.ascontiguousarray(a)).cuda()
qd = torch.from_numpy(np.ascontiguousarray(q)).cuda()
cfg = RefineConfig(precision="fp64", tol_factor=10.0 / n, max_iters=10)
ts = []
for r in range(reps + 2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    pair, rep = refine_template(ad, qd, cfg)
    torch.cuda.synchronize()
    if r >= 2:
        ts.append(time.perf_counter() - t0)
print("%.4f %.4f iters=%d" % (statistics.median(ts), min(ts), rep.iterations), flush=True)
