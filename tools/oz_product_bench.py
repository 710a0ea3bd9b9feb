"""One Ozaki-II hp product at size n (encode A^H, encode B, GEMM, decode) for profiling."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2203_10879_b200 import ZPlanar, ozaki  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
beta = int(sys.argv[2]) if len(sys.argv) > 2 else ozaki.HP_BETA
a = ZPlanar.from_any(torch.randn(n, n, dtype=torch.complex128))
b = ZPlanar.from_any(torch.randn(n, n, dtype=torch.complex128))
pl = ozaki.plan(n, beta, beta)
res = ozaki.ResidueBuffer(n, n, pl.nmod, "cuda")
ea = ozaki.encode(a, n, n, "a", pl, conj_t=True)
eb = ozaki.encode(b, n, n, "b", pl)
out = ZPlanar.empty(n)
for _ in range(2):
    ozaki.encode(a, n, n, "a", pl, conj_t=True, out=ea)
    ozaki.encode(b, n, n, "b", pl, out=eb)
    ozaki.gemm_residues(ea, eb, pl, res)
    ozaki.decode(res, ea, eb, pl, out)
torch.cuda.synchronize()
print("ok", n, pl.nmod)
