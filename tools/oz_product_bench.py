"""Phase timing of one Ozaki-II product at size n (encode A^H, encode B, GEMM,
decode), hp (FP64 in / out) and lp (complex64 in / out), CUDA events, median
of `reps`.  Usage: python tools/oz_product_bench.py [n] [reps]"""
import statistics
import sys

import torch

sys.path.insert(0, ".")
from paper_2203_10879_b200 import ZPlanar, ozaki  # noqa: E402
from paper_2203_10879_b200.matrix import lp_empty  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5


def run(tag, a, b, out, beta, gauss=False, herm=False):
    pl = ozaki.plan(n, beta, beta, gauss)
    res = ozaki.ResidueBuffer(n, n, pl.nmod, "cuda")
    ea = ozaki.encode(a, n, n, "a", pl, conj_t=True)
    eb = ozaki.encode(b, n, n, "b", pl)
    tag = ("G-" if gauss else "") + tag
    times = [[] for _ in range(4)]
    for rep in range(reps + 1):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
        ev[0].record()
        ozaki.encode(a, n, n, "a", pl, conj_t=True, out=ea)
        ev[1].record()
        ozaki.encode(b, n, n, "b", pl, out=eb)
        ev[2].record()
        ozaki.gemm_residues(ea, eb, pl, res, lower_only=herm)
        ev[3].record()
        ozaki.decode(res, ea, eb, pl, out, hermitian=herm)
        ev[4].record()
        torch.cuda.synchronize()
        if rep:
            for i in range(4):
                times[i].append(ev[i].elapsed_time(ev[i + 1]))
    t = [statistics.median(x) for x in times]
    if gauss:
        ops = 2.0 * (1 if herm else 2) * pl.nmod * n ** 3
    else:
        ops = 2.0 * (2 if eb.planes == 1 else 4) * pl.nmod * n ** 3 * (0.5 if herm else 1.0)
    print("%s n=%d nmod=%d: encA %.3f encB %.3f gemm %.3f (%.0f TOP/s) decode %.3f ms; total %.3f ms" % (
        tag, n, pl.nmod, t[0], t[1], t[2], ops / t[2] / 1e9, t[3], sum(t)), flush=True)


a = ZPlanar.from_any(torch.randn(n, n, dtype=torch.complex128))
b = ZPlanar.from_any(torch.randn(n, n, dtype=torch.complex128))
br = ZPlanar.from_any(torch.randn(n, n, dtype=torch.float64))
al, bl, ol = lp_empty(n), lp_empty(n), lp_empty(n)
al[:, :n] = torch.randn(n, n, dtype=torch.complex64)
bl[:, :n] = torch.randn(n, n, dtype=torch.complex64)
for g in (False, True):
    run("hp", a, b, ZPlanar.empty(n), ozaki.HP_BETA, g)
    run("hp-herm", a, a, ZPlanar.empty(n), ozaki.HP_BETA, g, herm=True)
    run("hp-realB", a, br, ZPlanar.empty(n), ozaki.HP_BETA, g)
    run("lp", al, bl, ol, ozaki.LP_BETA, g)
