"""Can the Gram product Y = Q^H Q - I run beside the lp solve?  Times, at
size n: the solve alone, the Hermitian hp product alone (encode, modular
GEMM, decode), and both on two streams with the GEMM's persistent grid
capped at `sms` SMs.  Usage: python tools/overlap_probe.py [n]"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2203_10879_b200 import ZPlanar, ozaki  # noqa: E402
from paper_2203_10879_b200.matrix import lp_empty  # noqa: E402
from paper_2203_10879_b200.trisolve import SolverWorkspace, solve_lp_device  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
g = torch.Generator(device="cuda").manual_seed(0)
t, e, l = lp_empty(n), lp_empty(n), lp_empty(n)
t[:, :n] = torch.triu(torch.randn(n, n, device="cuda", generator=g, dtype=torch.complex64))
t[:, :n].diagonal().copy_(torch.randn(n, device="cuda", generator=g, dtype=torch.complex64) * (n ** 0.5))
e[:, :n] = torch.tril(torch.randn(n, n, device="cuda", generator=g, dtype=torch.complex64), -1) * 1e-6
work = SolverWorkspace(n)
q = ZPlanar.from_any(torch.linalg.qr(torch.randn(n, n, dtype=torch.complex128, device="cuda", generator=g))[0])
y = ZPlanar.empty(n)
hp = ozaki.gauss_plan(n, ozaki.HP_BETA, ozaki.HP_BETA)
eb = ozaki.Encoded(n, n, 2, hp.beta_b, hp.nmod, "cuda")
res = ozaki.ResidueBuffer(n, n, hp.nmod, "cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def solve():
    solve_lp_device(t, e, l, n, None, work, torch.cuda.current_stream().cuda_stream)


def gram(sms):
    ozaki.encode(q, n, n, "b", hp, out=eb)  # Gaussian planes: one encoding for Q and Q^H
    ea = ozaki.conj_view(eb)
    ozaki.gemm_residues(ea, eb, hp, res, lower_only=True, num_sms=sms)
    ozaki.decode(res, ea, eb, hp, y, shift=-1.0, hermitian=True)


def timed(fn, reps=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def both(sms):
    main = torch.cuda.current_stream()
    s1.wait_stream(main)
    s2.wait_stream(main)
    with torch.cuda.stream(s1):
        solve()
    with torch.cuda.stream(s2):
        gram(sms)
    main.wait_stream(s1)
    main.wait_stream(s2)


ts = timed(solve)
print("n=%d solve alone %.2f ms" % (n, ts), flush=True)
for sms in (148, 128, 112, 96, 72):
    tg = timed(lambda: gram(sms))
    tb = timed(lambda: both(sms))
    print("gram on %3d SMs alone %.2f ms; solve + gram concurrently %.2f ms (sequential %.2f)" % (
        sms, tg, tb, ts + tg), flush=True)
