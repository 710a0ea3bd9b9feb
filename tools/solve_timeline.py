"""Kernel timeline of one lp triangular solve (graph replay) at size n.

Needs the diagnostic build of the library with -DSR_TIMELINE (per-kernel
%globaltimer start / end marks; compiled out of libsr.so):
  for f in paper_2203_10879_b200/csrc/*.cu; do nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
    -Xcompiler -fPIC --expt-relaxed-constexpr -DSR_TIMELINE -c $f -o tools/_ab/tl/$(basename $f .cu).o; done
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o tools/_ab/libsr_tl.so tools/_ab/tl/*.o
Usage: python tools/solve_timeline.py [n] [lib]"""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2203_10879_b200.matrix import lp_empty  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
lib = ctypes.CDLL(sys.argv[2] if len(sys.argv) > 2 else "tools/_ab/libsr_tl.so")
P = ctypes.c_void_p
lib.sr_trisolve_workspace_bytes.restype = ctypes.c_size_t
lib.sr_trisolve_workspace_bytes.argtypes = [ctypes.c_int, ctypes.c_int]
lib.sr_trisolve_c64.argtypes = [ctypes.c_int, P, P, ctypes.c_longlong, P, ctypes.c_float, P, P, P, ctypes.c_size_t, P]
for f in (lib.sr_timeline_solve, lib.sr_timeline_tc):
    f.argtypes = [P, ctypes.c_int]

g = torch.Generator(device="cuda").manual_seed(0)
t, e, l = lp_empty(n), lp_empty(n), lp_empty(n)
t[:, :n] = torch.triu(torch.randn(n, n, device="cuda", generator=g, dtype=torch.complex64))
t[:, :n].diagonal().copy_(torch.randn(n, device="cuda", generator=g, dtype=torch.complex64) * (n ** 0.5))
e[:, :n] = torch.tril(torch.randn(n, n, device="cuda", generator=g, dtype=torch.complex64), -1) * 1e-6
wsb = lib.sr_trisolve_workspace_bytes(n, 1)
ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
clipped = torch.zeros(1, dtype=torch.int64, device="cuda")
flags = torch.zeros(1, dtype=torch.int32, device="cuda")
st = torch.cuda.current_stream().cuda_stream


def solve():
    rc = lib.sr_trisolve_c64(n, t.data_ptr(), e.data_ptr(), t.shape[1], l.data_ptr(), 0.0, clipped.data_ptr(),
                             flags.data_ptr(), ws.data_ptr(), wsb, st)
    assert rc == 0, rc


for _ in range(3):
    solve()
torch.cuda.synchronize()
lib.sr_timeline_solve(None, 1)
lib.sr_timeline_tc(None, 1)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
solve()
e1.record()
torch.cuda.synchronize()
a = np.zeros((8, 1024, 2), dtype=np.uint64)
b = np.zeros((8, 1024, 2), dtype=np.uint64)
lib.sr_timeline_solve(a.ctypes.data, 0)
lib.sr_timeline_tc(b.ctypes.data, 0)
tl = np.where(a[:, :, 0] == np.uint64(2 ** 64 - 1), 0, 1)
N = (n + 31) // 32
t0 = int(a[0, 0, 0])


def span(arr, k, s):
    st_, en = int(arr[k, s, 0]), int(arr[k, s, 1])
    if st_ == 2 ** 64 - 1 or en == 0:
        return None
    return (st_ - t0) / 1e3, (en - t0) / 1e3


print("n=%d levels=%d event time %.3f ms; timeline span %.3f ms" % (
    n, N, e0.elapsed_time(e1), (int(a[0, N - 1, 1]) - t0) / 1e6))
sd, gaps, nd = [], [], []
for lev in range(N):
    s = span(a, 0, lev)
    if s:
        sd.append(s[1] - s[0])
    if lev:
        p = span(a, 0, lev - 1)
        if s and p:
            gaps.append(s[0] - p[1])
    q = span(a, 1, lev)
    if q:
        nd.append(q[1] - q[0])
print("SOLVE: mean %.1f us, median %.1f, max %.1f; gap SOLVE(l-1) end -> SOLVE(l) start: mean %.1f us, median %.1f, "
      "max %.1f" % (np.mean(sd), np.median(sd), np.max(sd), np.mean(gaps), np.median(gaps), np.max(gaps)))
print("NEAR: mean %.1f us, median %.1f, max %.1f" % (np.mean(nd), np.median(nd), np.max(nd)))
fd = {2: [], 3: [], 4: [], 5: []}
for k in fd:
    for bb in range(N // 4 + 1):
        s = span(b, k, bb)
        if s:
            fd[k].append(s[1] - s[0])
for k, name in ((2, "far COL"), (3, "far ROW"), (4, "lforms"), (5, "lmax")):
    if fd[k]:
        print("%s: %d launches, mean %.1f us, total %.1f us" % (name, len(fd[k]), np.mean(fd[k]), np.sum(fd[k])))
print("level  solve[start,end]  near[start,end]  (us from the first SOLVE start); far batches at batch ends")
for lev in list(range(0, 12)) + list(range(N // 2, N // 2 + 8)) + list(range(N - 6, N)):
    s, q = span(a, 0, lev), span(a, 1, lev)
    line = "%4d  %s  %s" % (lev, "[%9.1f,%9.1f]" % s if s else "-", "[%9.1f,%9.1f]" % q if q else "-")
    if lev % 4 == 3:
        bb = lev // 4
        for k, nm in ((5, "lmax"), (4, "lform"), (2, "COL"), (3, "ROW")):
            f = span(b, k, bb)
            if f:
                line += "  %s[%.1f,%.1f]" % (nm, f[0], f[1])
    print(line)
