"""Where the end-to-end time goes: refine_template from pinned host memory
(H2D of A and Q^, D2H of Q and T inside) against the same call on
device-resident inputs, with host timestamps at every phase mark.
Usage: python tools/e2e_probe.py [n] [reps]"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2203_10879_b200 import RefineConfig, ZPlanar, inputs, refine  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
a_np = inputs.gaussian_real(n, 0)
q_np = inputs.cached_qhat("c3_n%d_s0" % n, a_np).astype(np.complex128)
cfg = RefineConfig(precision="fp64", tol_factor=10.0 / n, max_iters=10)
dev = torch.device("cuda", 0)
A = ZPlanar.from_any(a_np, device=dev)
Q = ZPlanar.from_any(q_np, device=dev)
a_host = torch.from_numpy(a_np).pin_memory()
q_host = torch.from_numpy(q_np).pin_memory()
q_out = torch.empty((n, n), dtype=torch.complex128).pin_memory()
t_out = torch.empty((n, n), dtype=torch.complex128).pin_memory()

host_marks = []
_orig = refine._mark


def mark(label):
    torch.cuda.current_stream().synchronize() if SYNC else None
    host_marks.append((label, time.perf_counter()))
    _orig(label)


refine._mark = mark
SYNC = False


def timed(fn, tag):
    global host_marks
    torch.cuda.synchronize()
    host_marks = []
    refine.PHASES = []
    t0 = time.perf_counter()
    fn()
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    ph = refine.PHASES
    refine.PHASES = None
    dev_ms = ph[0][1].elapsed_time(ph[-1][1]) if len(ph) > 1 else float("nan")
    first = host_marks[0][1] - t0 if host_marks else float("nan")
    last = t1 - host_marks[-1][1] if host_marks else float("nan")
    print("%-10s wall %.1f ms | host before first mark %.1f ms | device start->last mark %.1f ms | after last "
          "mark %.1f ms" % (tag, (t1 - t0) * 1e3, first * 1e3, dev_ms, last * 1e3), flush=True)
    if tag.startswith("host") and VERBOSE:
        prev = t0
        for (lab, t), (_, ev) in zip(host_marks, ph):
            print("    %-12s host +%.1f ms" % (lab, (t - prev) * 1e3))
            prev = t


VERBOSE = False
for _ in range(2):
    refine.refine_template(A, Q, cfg, device=dev)
    refine.refine_template(a_host, q_host, cfg, device=dev, out=(q_out, t_out))
for r in range(reps):
    VERBOSE = r == reps - 1
    timed(lambda: refine.refine_template(A, Q, cfg, device=dev), "device")
    timed(lambda: refine.refine_template(a_host, q_host, cfg, device=dev, out=(q_out, t_out)), "host-io")
    timed(lambda: refine.refine_template(A, Q, cfg, device=dev, out=(q_out, t_out)), "dev-in/host-out")
    timed(lambda: refine.refine_template(a_host, q_host, cfg, device=dev), "host-in")
# raw copy rates
for nbytes in (1 << 30,):
    h = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    d = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    for tag, fn in (("H2D", lambda: d.copy_(h, non_blocking=True)), ("D2H", lambda: h.copy_(d, non_blocking=True))):
        fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        print("%s 1 GiB pinned: %.1f ms (%.1f GB/s)" % (tag, dt * 1e3, nbytes / dt / 1e9))

# ---- host-path breakdown (wrappers with a device sync on both sides)
def wrap(name):
    f = getattr(refine, name)

    def g(*a, **k):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = f(*a, **k)
        torch.cuda.synchronize()
        print("    %-14s %.1f ms" % (name, (time.perf_counter() - t0) * 1e3), flush=True)
        return r
    setattr(refine, name, g)


for name in ("_upload_qhat", "_AsyncUpload", "_workspace", "_HostResult", "_coerce"):
    wrap(name)
timed(lambda: refine.refine_template(a_host, q_host, cfg, device=dev, out=(q_out, t_out)), "host-io")
timed(lambda: refine.refine_template(a_host, q_host, cfg, device=dev), "host-in")
