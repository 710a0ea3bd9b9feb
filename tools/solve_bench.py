"""Time the lp triangular solver alone: stril(T L - L T) = -E at size n."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2203_10879_b200.matrix import lp_empty  # noqa: E402
from paper_2203_10879_b200.trisolve import SolverWorkspace, solve_lp_device  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
g = torch.Generator(device="cuda").manual_seed(0)
t = lp_empty(n)
e = lp_empty(n)
l = lp_empty(n)
tr = torch.randn(n, n, device="cuda", generator=g, dtype=torch.complex64)
t[:, :n] = torch.triu(tr)
d = torch.randn(n, device="cuda", generator=g, dtype=torch.complex64) * (n ** 0.5)
t[:, :n].diagonal().copy_(d)
e[:, :n] = torch.tril(torch.randn(n, n, device="cuda", generator=g, dtype=torch.complex64), -1) * 1e-6
work = SolverWorkspace(n)
st = torch.cuda.current_stream().cuda_stream
for _ in range(2):
    solve_lp_device(t, e, l, n, None, work, st)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    solve_lp_device(t, e, l, n, None, work, st)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
print("trisolve n=%d: %.2f ms per solve (%.1f GFLOP/s useful, n^3/3 cmac)" % (n, ms, 8 * n ** 3 / 3 / ms / 1e6))
if len(sys.argv) > 3:  # every solve from an idle GPU (as inside a refinement): event and host times
    for _ in range(reps):
        torch.cuda.synchronize()
        h0 = time.perf_counter()
        e0.record()
        solve_lp_device(t, e, l, n, None, work, st)
        h1 = time.perf_counter()
        e1.record()
        torch.cuda.synchronize()
        print("  isolated solve: %.2f ms on the device, host enqueue %.2f ms" % (e0.elapsed_time(e1), (h1 - h0) * 1e3))
lv = l[:, :n]
res = torch.linalg.matrix_norm(torch.tril(t[:, :n].to(torch.complex128) @ lv.to(torch.complex128)
                               - lv.to(torch.complex128) @ t[:, :n].to(torch.complex128), -1)
                               + e[:, :n].to(torch.complex128)) / torch.linalg.matrix_norm(e[:, :n].to(torch.complex128))
print("relative residual %.3e" % float(res))
