"""Interleaved A/B of the modular GEMM with and without wide (N = 512) units
(SR_OZ_WIDE, read at every launch): Gaussian hp complex, complex x real and
Hermitian products at n = 8192, median of the interleaved repetitions."""
import os
import statistics
import sys

import torch

sys.path.insert(0, ".")
from paper_2203_10879_b200 import ZPlanar, ozaki  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 7
g = torch.Generator(device="cuda").manual_seed(0)
q = ZPlanar.from_any(torch.randn(n, n, dtype=torch.complex128, device="cuda", generator=g))
a = ZPlanar.from_any(torch.randn(n, n, dtype=torch.float64, device="cuda", generator=g))
pl = ozaki.gauss_plan(n, ozaki.HP_BETA, ozaki.HP_BETA)
eq = ozaki.encode(q, n, n, "b", pl)
ea = ozaki.encode(a, n, n, "b", pl)
res = ozaki.ResidueBuffer(n, n, pl.nmod, "cuda")
cases = {"complex": (ozaki.conj_view(eq), eq, False), "cplx_x_real": (ozaki.conj_view(eq), ea, False),
         "hermitian": (ozaki.conj_view(eq), eq, True)}
times = {(c, w): [] for c in cases for w in (0, 1)}
for r in range(reps):
    for c, (x, y, herm) in cases.items():
        for w in (0, 1):
            os.environ["SR_OZ_WIDE"] = str(w)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            ozaki.gemm_residues(x, y, pl, res, lower_only=herm)
            e1.record()
            torch.cuda.synchronize()
            if r:
                times[(c, w)].append(e0.elapsed_time(e1))
for c in cases:
    t0, t1 = statistics.median(times[(c, 0)]), statistics.median(times[(c, 1)])
    print("%-12s n=%d: narrow %.3f ms  wide %.3f ms  (%.1f %%)" % (c, n, t0, t1, 100 * (t1 / t0 - 1)), flush=True)
