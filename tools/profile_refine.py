"""One config-3 refinement inside cudaProfilerStart/Stop, for
    ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
        --log-file launches.csv python tools/profile_refine.py [n]
(one warm-up refinement runs outside the profiled range).  Prints the result."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2203_10879_b200 import RefineConfig, inputs, refine_template  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
a, q = inputs.config_inputs(3, n=n)
ad = torch.from_numpy(np.ascontiguousarray(a)).cuda()
qd = torch.from_numpy(np.ascontiguousarray(q)).cuda()
cfg = RefineConfig(precision="fp64", tol_factor=10.0 / n, max_iters=10)
refine_template(ad, qd, cfg)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
pair, rep = refine_template(ad, qd, cfg)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("n=%d status %s iterations %d" % (n, rep.status.value, rep.iterations), flush=True)
