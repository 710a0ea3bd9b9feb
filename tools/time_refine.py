"""Quick timing of refine_template (FP64 mode) and its GEMM on one GPU."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2203_10879_b200 import RefineConfig, ZPlanar, inputs, matmul_hp, refine_template  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
rng = np.random.default_rng(0)
# GEMM throughput
a = ZPlanar.from_any(torch.randn(n, n, dtype=torch.complex128))
b = ZPlanar.from_any(torch.randn(n, n, dtype=torch.complex128))
br = ZPlanar.from_any(torch.randn(n, n, dtype=torch.float64))
c = ZPlanar.empty(n)
for trans, bb, flops, name in ((False, b, 8, "NN"), (True, b, 8, "CN"), (True, br, 4, "CN-real")):
    for _ in range(2):
        matmul_hp(a, bb, trans_a=trans, out=c)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    reps = 5
    for _ in range(reps):
        matmul_hp(a, bb, trans_a=trans, out=c)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print("zgemm %s n=%d: %.3f ms  %.2f TFLOP/s" % (name, n, ms, flops * n ** 3 / ms / 1e9), flush=True)

from paper_2203_10879_b200 import ozaki  # noqa: E402
for beta, tag in ((ozaki.HP_BETA, "hp"), (ozaki.LP_BETA, "lp")):
    pl = ozaki.plan(n, beta, beta)
    res = ozaki.ResidueBuffer(n, n, pl.nmod, "cuda")
    ea = ozaki.encode(a, n, n, "a", pl, conj_t=True)
    eb = ozaki.encode(b, n, n, "b", pl)
    out = ZPlanar.empty(n)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
    for rep in range(3):
        ev[0].record()
        ozaki.encode(a, n, n, "a", pl, conj_t=True, out=ea)
        ev[1].record()
        ozaki.encode(b, n, n, "b", pl, out=eb)
        ev[2].record()
        ozaki.gemm_residues(ea, eb, pl, res)
        ev[3].record()
        ozaki.decode(res, ea, eb, pl, out)
        ev[4].record()
        torch.cuda.synchronize()
    t = [ev[i].elapsed_time(ev[i + 1]) for i in range(4)]
    g_ops = 2.0 * 4 * pl.nmod * n ** 3
    print("ozaki %s n=%d nmod=%d: encA %.3f encB %.3f gemm %.3f ms (%.0f TOP/s int8, %.1f TF/s fp64-equiv) "
          "decode %.3f ms; total %.3f ms" % (tag, n, pl.nmod, t[0], t[1], t[2], g_ops / t[2] / 1e9,
                                            8 * n ** 3 / t[2] / 1e9, t[3], sum(t)), flush=True)

if n <= 4096:
    A = inputs.gaussian_complex(n, 0)
    Q = inputs.schur_vectors(A).astype(np.complex128)
    for gemm in ("ozaki", "dmma"):
      cfg = RefineConfig(precision="fp64", tol_factor=10.0 / n, max_iters=10, gemm=gemm)
      for rep in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        pair, r = refine_template(A, Q, cfg)
        torch.cuda.synchronize()
        print("refine[%s] n=%d: %.3f s  status %s it %d hist %s" % (
            gemm, n, time.perf_counter() - t0, r.status.value, r.iterations,
            ["%.2e" % (h[0] / np.linalg.norm(A)) for h in r.residual_history]), flush=True)

# Q^ generation options at large n (setup only): LAPACK cgees vs GPU eig + QR
if len(sys.argv) > 2 and int(sys.argv[2]) > 0:
    import scipy.linalg
    m = int(sys.argv[2])
    A = inputs.gaussian_real(m, 0)
    t0 = time.perf_counter()
    try:
        w, v = torch.linalg.eig(torch.from_numpy(A).to(torch.complex64).cuda())
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        q, _ = torch.linalg.qr(v)
        torch.cuda.synchronize()
        qn = q.cpu().numpy().astype(np.complex128)
        th = (qn.conj().T @ A) @ qn
        print("gpu eig+qr n=%d: eig %.1fs qr %.1fs relE %.2e ortho %.2e" % (
            m, t1 - t0, time.perf_counter() - t1, np.linalg.norm(np.tril(th, -1)) / np.linalg.norm(A),
            np.linalg.norm(qn.conj().T @ qn - np.eye(m))), flush=True)
    except Exception as ex:
        print("gpu eig failed:", ex, flush=True)
    t0 = time.perf_counter()
    _, z = scipy.linalg.schur(A.astype(np.complex64), output="complex")
    zq = z.astype(np.complex128)
    th = (zq.conj().T @ A) @ zq
    print("cgees n=%d: %.1fs relE %.2e ortho %.2e" % (m, time.perf_counter() - t0,
          np.linalg.norm(np.tril(th, -1)) / np.linalg.norm(A),
          np.linalg.norm(zq.conj().T @ zq - np.eye(m))), flush=True)


def phase_profile(A, Q, cfg, label):
    import collections
    from paper_2203_10879_b200 import refine as R
    refine_template(A, Q, cfg)
    torch.cuda.synchronize()
    R.PHASES = []
    t0 = time.perf_counter()
    pair, r = refine_template(A, Q, cfg)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    ph, R.PHASES = R.PHASES, None
    acc = collections.OrderedDict()
    for (l0, e0), (l1, e1) in zip(ph, ph[1:]):
        acc[l1] = acc.get(l1, 0.0) + e0.elapsed_time(e1)
    print("phases[%s] n=%d wall %.3f s, iterations %d: %s" % (label, A.shape[0] if hasattr(A, "shape") else 0,
          wall, r.iterations, ", ".join("%s %.1f ms" % kv for kv in acc.items())), flush=True)
    print("  history relE:", ["%.2e" % (h[0] / float(np.linalg.norm(A))) for h in r.residual_history], flush=True)


if len(sys.argv) > 3:
    m = int(sys.argv[3])
    Am = inputs.gaussian_real(m, 0)
    Qm = inputs.cached_qhat("c3_n%d_s0" % m, Am).astype(np.complex128)
    phase_profile(Am, Qm, RefineConfig(precision="fp64", tol_factor=10.0 / m, max_iters=10), "ozaki")
