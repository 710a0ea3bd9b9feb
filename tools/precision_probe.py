"""Measurement noise of the FP64 products vs an exact (double-double) oracle:
||stril((Q^H A) Q) - exact||_F / ||A||_F and ||(Q^H Q - I) - exact||_F in
units of u64, for numpy (OpenBLAS) and the libsr DMMA kernel."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import clib  # noqa: E402
from paper_2203_10879_b200 import ZPlanar, matmul_hp, ozaki  # noqa: E402


import os  # noqa: E402
BETAS = [int(b) for b in os.environ.get("OZ_BETAS", str(ozaki.HP_BETA)).split(",")]


def oz(x, y, trans=False, shift=0.0, beta=None):
    beta = ozaki.HP_BETA if beta is None else beta
    pl = ozaki.plan(x.rows, beta, beta)
    ea = ozaki.encode(x, x.rows, x.cols, "a", pl, conj_t=trans)
    eb = ozaki.encode(y, y.rows, y.cols, "b", pl)
    res = ozaki.ResidueBuffer(x.cols if trans else x.rows, y.cols, pl.nmod, "cuda")
    ozaki.gemm_residues(ea, eb, pl, res)
    out = ZPlanar.empty(res.M, res.N)
    ozaki.decode(res, ea, eb, pl, out, shift=shift)
    return out

U = 2.0 ** -53


def dd_planes(x):
    z = np.zeros(x.shape)
    return (np.ascontiguousarray(x.real), z, np.ascontiguousarray(x.imag), z.copy())


def dd_gemm(a_planes, b_planes):
    return clib.gemm_dd(a_planes, b_planes)


def conj_t(p):
    return tuple(np.ascontiguousarray(x.T) * (1 if i < 2 else -1) for i, x in enumerate(p))


for n in [int(x) for x in sys.argv[1:]] or [256, 512]:
    rng = np.random.default_rng(n)
    a = (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))) * np.sqrt(0.5)
    z = (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)))
    q, r = np.linalg.qr(z)
    qp, ap = dd_planes(q), dd_planes(a)
    p_ex = dd_gemm(conj_t(qp), ap)
    t_ex = dd_gemm(p_ex, qp)
    g_ex = dd_gemm(conj_t(qp), qp)
    t_hi = (t_ex[0] + 1j * t_ex[2]) + (t_ex[1] + 1j * t_ex[3])
    g_lo = (g_ex[0] - np.eye(n)) + g_ex[1] + 1j * (g_ex[2] + g_ex[3])
    na = np.linalg.norm(a)
    t_np = (q.conj().T @ a) @ q
    g_np = q.conj().T @ q - np.eye(n)
    qd, ad = ZPlanar.from_any(q), ZPlanar.from_any(a)
    t_gpu = matmul_hp(matmul_hp(qd, ad, trans_a=True), qd).to_numpy()
    g_gpu = matmul_hp(qd, qd, trans_a=True, diag_shift=-1.0).to_numpy()
    rows = [("numpy", t_np, g_np), ("dmma", t_gpu, g_gpu)]
    for beta in BETAS:
        t_oz = oz(oz(qd, ad, trans=True, beta=beta), qd, beta=beta).to_numpy()
        g_oz = oz(qd, qd, trans=True, shift=-1.0, beta=beta).to_numpy()
        rows.append(("oz%d/%d" % (beta, ozaki.plan(n, beta, beta).nmod), t_oz, g_oz))
    for name, t, g in rows:
        et = np.linalg.norm(np.tril(t - t_hi, -1)) / na / U
        eg = np.linalg.norm(g - g_lo) / U
        print("n=%d %-9s stril(T) noise %.2f u*||A||   Y noise %.2f u  (true ||Y|| %.2f u)" % (
            n, name, et, eg, np.linalg.norm(g_lo) / U), flush=True)
