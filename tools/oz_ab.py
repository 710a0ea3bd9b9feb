"""In-process A/B of oz_gemm variants (cluster vs none, group sizes) at n=8192, interleaved."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2203_10879_b200 import ZPlanar, ozaki  # noqa: E402

n = 8192
a = ZPlanar.from_any(torch.randn(n, n, dtype=torch.complex128))
b = ZPlanar.from_any(torch.randn(n, n, dtype=torch.complex128))
pl = ozaki.plan(n, ozaki.HP_BETA, ozaki.HP_BETA)
res = ozaki.ResidueBuffer(n, n, pl.nmod, "cuda")
ea = ozaki.encode(a, n, n, "a", pl, conj_t=True)
eb = ozaki.encode(b, n, n, "b", pl)
variants = {"cluster_g8": {"SR_OZ_GROUP_M": "8"}, "cluster_g16": {"SR_OZ_GROUP_M": "16"},
            "nocluster_g16": {"SR_OZ_NO_CLUSTER": "1", "SR_OZ_GROUP_M": "16"},
            "nocluster_g8": {"SR_OZ_NO_CLUSTER": "1", "SR_OZ_GROUP_M": "8"}}
times = {k: [] for k in variants}
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for rnd in range(6):
    for name, env in variants.items():
        for k in ("SR_OZ_NO_CLUSTER", "SR_OZ_GROUP_M"):
            os.environ.pop(k, None)
        os.environ.update(env)
        ozaki.gemm_residues(ea, eb, pl, res)
        e0.record()
        ozaki.gemm_residues(ea, eb, pl, res)
        e1.record()
        torch.cuda.synchronize()
        times[name].append(e0.elapsed_time(e1))
ops = 2.0 * 4 * pl.nmod * n ** 3
for name, t in times.items():
    m = float(np.median(t))
    print("%-15s median %.2f ms  (%.0f TOP/s)  all %s" % (name, m, ops / m / 1e9, ["%.1f" % x for x in t]))
