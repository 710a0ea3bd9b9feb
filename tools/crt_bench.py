"""Encode / decode timing of the Gaussian Ozaki-II products at size n (CUDA
events, median of reps): the SIMT and tensor-core CRT decodes on the same
residues (sr_oz_config key 0), hp complex, hp Hermitian and lp.
Usage: python tools/crt_bench.py [n] [reps]"""
import statistics
import sys

import torch

sys.path.insert(0, ".")
from paper_2203_10879_b200 import ZPlanar, _lib, ozaki  # noqa: E402
from paper_2203_10879_b200.matrix import lp_empty  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
lib = _lib.load()


def timed(fn):
    ts = []
    for rep in range(reps + 1):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        if rep:
            ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


def case(tag, a, b, out, beta, herm=False, conj=True, add=None):
    pl = ozaki.plan(n, beta, beta, gauss=True)
    res = ozaki.ResidueBuffer(n, n, pl.nmod, "cuda")
    if herm:
        eb = ozaki.encode(b, n, n, "b", pl)
        ea = ozaki.conj_view(eb)
    else:
        ea = ozaki.encode(a, n, n, "a", pl, conj_t=conj)
        eb = ozaki.encode(b, n, n, "b", pl)
    t_ea = timed(lambda: ozaki.encode(a, n, n, "a", pl, conj_t=conj, out=ea)) if not herm else 0.0
    t_eb = timed(lambda: ozaki.encode(b, n, n, "b", pl, out=eb))
    ozaki.gemm_residues(ea, eb, pl, res, lower_only=herm)
    t = {}
    for mode in (0, 1):
        lib.sr_oz_config(0, mode)
        t[mode] = timed(lambda: ozaki.decode(res, ea, eb, pl, out, hermitian=herm, add=add,
                                             alpha=0.5 if add is not None else 1.0))
    lib.sr_oz_config(0, 1)
    nb = 2 * pl.nmod * n * n
    print("%-10s n=%d nmod=%d chunks=%d: encA %.3f encB %.3f ms | decode SIMT %.3f  TC %.3f ms (%.2fx; residues %.2f GB)"
          % (tag, n, pl.nmod, pl.decode_chunks(24 if isinstance(out, torch.Tensor) else 53), t_ea, t_eb, t[0], t[1],
             t[0] / t[1], nb / 1e9), flush=True)


g = torch.Generator().manual_seed(0)
a = ZPlanar.from_any(torch.randn(n, n, generator=g, dtype=torch.complex128).cuda())
b = ZPlanar.from_any(torch.randn(n, n, generator=g, dtype=torch.complex128).cuda())
out = ZPlanar.empty(n)
case("hp", a, b, out, ozaki.HP_BETA)
case("hp+add", a, b, out, ozaki.HP_BETA, add=a)
case("hp-herm", a, b, out, ozaki.HP_BETA_Q, herm=True)
al, bl, ol = lp_empty(n), lp_empty(n), lp_empty(n)
al[:, :n] = torch.randn(n, n, generator=g, dtype=torch.complex64).cuda()
bl[:, :n] = torch.randn(n, n, generator=g, dtype=torch.complex64).cuda()
case("lp", al, bl, ol, ozaki.LP_BETA, conj=False)
