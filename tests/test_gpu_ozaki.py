"""GPU parity of the Ozaki-II int8 tensor-core products.

1. The tcgen05 modular GEMM is checked bit-exactly against numpy integer
   arithmetic (integer work: the bar is bit-exact).
2. The emulated FP64 products are checked against an exact double-double
   evaluation (oracle/ddgemm_oracle.c, the reference's gemm_hp restated): the
   Ozaki result must be at least as accurate as numpy's FP64 BLAS product.
"""
import numpy as np
import pytest
import torch

from oracle import clib
from paper_2203_10879_b200 import ZPlanar, _lib, ozaki
from paper_2203_10879_b200.matrix import lp_empty

pytestmark = pytest.mark.gpu


def sym_residues(rng, shape, p):
    lo, hi = -(p // 2), (p + 1) // 2 - 1
    return rng.integers(lo, hi + 1, size=shape).astype(np.int8)


def sym_mod(x, p):
    r = np.mod(x, p)
    hi = (p + 1) // 2 - 1
    return np.where(r > hi, r - p, r)


@pytest.mark.parametrize("M,N,K,cplx", [(128, 128, 64, True), (200, 130, 100, True), (256, 384, 512, True),
                                        (77, 300, 1000, False), (129, 129, 129, True)])
def test_oz_gemm_residues_bit_exact(M, N, K, cplx):
    rng = np.random.default_rng(M + N + K)
    moduli = [256, 255, 253]
    kp = ozaki.kpitch(K)
    bp = 3 if cplx else 1
    a = np.zeros((len(moduli), 2, M, kp), np.int8)
    b = np.zeros((len(moduli), bp, N, kp), np.int8)
    for l, p in enumerate(moduli):
        a[l, :, :, :K] = sym_residues(rng, (2, M, K), p)
        if cplx:
            re = sym_residues(rng, (N, K), p)
            im = sym_residues(rng, (N, K), p)
            b[l, 0, :, :K] = sym_mod(-im.astype(np.int64), p)
            b[l, 1, :, :K] = re
            b[l, 2, :, :K] = im
        else:
            b[l, 0, :, :K] = sym_residues(rng, (N, K), p)
    ad, bd = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    pitch = ozaki.kpitch(N)
    out = torch.zeros((len(moduli), 2, M, pitch), dtype=torch.int8, device="cuda")
    mods = np.array(moduli, np.int32)
    _lib.call("sr_oz_gemm_i8", M, N, K, len(moduli), mods.ctypes.data, ad.data_ptr(), 2, kp, bd.data_ptr(), bp,
              kp, out.data_ptr(), pitch, 0, 0, torch.cuda.current_stream().cuda_stream)
    got = out.cpu().numpy()[:, :, :, :N].astype(np.int64)
    for l, p in enumerate(moduli):
        ar, ai = a[l, 0].astype(np.int64), a[l, 1].astype(np.int64)
        if cplx:
            br, bi = b[l, 1].astype(np.int64), b[l, 2].astype(np.int64)
            cre = ar @ br.T - ai @ bi.T
            cim = ar @ bi.T + ai @ br.T
        else:
            br = b[l, 0].astype(np.int64)
            cre, cim = ar @ br.T, ai @ br.T
        assert np.array_equal(got[l, 0], sym_mod(cre, p)), (l, p)
        assert np.array_equal(got[l, 1], sym_mod(cim, p)), (l, p)


def dd_exact(a, b):
    z = np.zeros(a.shape)
    pa = (np.ascontiguousarray(a.real), z, np.ascontiguousarray(a.imag), z.copy())
    z = np.zeros(b.shape)
    pb = (np.ascontiguousarray(b.real), z, np.ascontiguousarray(np.imag(b)), z.copy())
    o = clib.gemm_dd(pa, pb)
    return (o[0] + o[1]) + 1j * (o[2] + o[3]), o


def oz_product(x, y, trans=False, alpha=1.0, shift=0.0, beta=ozaki.HP_BETA, hermitian=False):
    xm, ym = ZPlanar.from_any(x), ZPlanar.from_any(y)
    K = x.shape[0] if trans else x.shape[1]
    M = x.shape[1] if trans else x.shape[0]
    N = y.shape[1]
    pl = ozaki.plan(K, beta, beta)
    ea = ozaki.encode(xm, x.shape[0], x.shape[1], "a", pl, conj_t=trans)
    eb = ozaki.encode(ym, y.shape[0], y.shape[1], "b", pl)
    res = ozaki.ResidueBuffer(M, N, pl.nmod, "cuda")
    ozaki.gemm_residues(ea, eb, pl, res, lower_only=hermitian)
    out = ZPlanar.empty(M, N)
    ozaki.decode(res, ea, eb, pl, out, alpha=alpha, shift=shift, hermitian=hermitian)
    return out.to_numpy()


@pytest.mark.parametrize("M,N,K", [(1, 1, 1), (64, 48, 40), (200, 130, 257), (256, 256, 256)])
@pytest.mark.parametrize("trans", [False, True])
@pytest.mark.parametrize("b_real", [False, True])
def test_oz_fp64_product_beats_blas(M, N, K, trans, b_real):
    rng = np.random.default_rng(M * 7 + N + K)
    x = rng.standard_normal((K, M) if trans else (M, K)) + 1j * rng.standard_normal((K, M) if trans else (M, K))
    y = rng.standard_normal((K, N))
    if not b_real:
        y = y + 1j * rng.standard_normal((K, N))
    xo = x.conj().T if trans else x
    exact, _ = dd_exact(xo, y)
    got = oz_product(x, y, trans=trans)
    blas = xo @ y
    e_oz = np.linalg.norm(got - exact)
    e_blas = np.linalg.norm(blas - exact)
    scale = np.linalg.norm(exact)
    assert e_oz <= max(2 * e_blas, 4 * 2.0 ** -53 * scale), (e_oz / scale, e_blas / scale)


@pytest.mark.parametrize("n,hermitian", [(200, False), (200, True), (300, True)])
def test_oz_gram_minus_identity_is_accurate(n, hermitian):
    rng = np.random.default_rng(3)
    q, _ = np.linalg.qr(rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)))
    _, o = dd_exact(q.conj().T, q)
    exact = (o[0] - np.eye(n)) + o[1] + 1j * (o[2] + o[3])
    got = oz_product(q, q, trans=True, shift=-1.0, hermitian=hermitian)
    blas = q.conj().T @ q - np.eye(n)
    if hermitian:
        assert np.array_equal(got, got.conj().T)
    assert np.linalg.norm(got - exact) <= np.linalg.norm(blas - exact)


def test_oz_lp_product_complex64():
    rng = np.random.default_rng(9)
    n = 300
    w = ((rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))) * 1e-3).astype(np.complex64)
    wd = lp_empty(n)
    wd[:, :n] = torch.from_numpy(w)
    pl = ozaki.plan(n, ozaki.LP_BETA, ozaki.LP_BETA)
    ea = ozaki.encode(wd, n, n, "a", pl)
    eb = ozaki.encode(wd, n, n, "b", pl)
    res = ozaki.ResidueBuffer(n, n, pl.nmod, "cuda")
    ozaki.gemm_residues(ea, eb, pl, res)
    out = lp_empty(n)
    ozaki.decode(res, ea, eb, pl, out)
    ref = w.astype(np.complex128) @ w.astype(np.complex128)
    got = out[:, :n].cpu().numpy()
    err = np.linalg.norm(got - ref) / np.linalg.norm(ref)
    f32 = np.linalg.norm((w @ w) - ref) / np.linalg.norm(ref)
    assert err <= max(2 * f32, 1e-7), (err, f32)


@pytest.mark.parametrize("dtype,beta", [(torch.complex64, ozaki.LP_BETA), (torch.complex128, ozaki.DD_LP_BETA)])
@pytest.mark.parametrize("n", [300, 515])
def test_oz_lp_structured_products(dtype, beta, n):
    """W = L - L^H skew-Hermitian: W^2 (Hermitian) and W^3 = W^2 W (skew) from
    the lower 128-tiles plus the mirror; upper tiles exactly (-)conj of the
    lower ones, accuracy as the full product."""
    rng = np.random.default_rng(n)
    npdt = np.complex64 if dtype == torch.complex64 else np.complex128
    l = np.tril(rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)), -1) * 1e-3
    w = (l - l.conj().T).astype(npdt)
    wd = lp_empty(n, dtype=dtype)
    wd[:, :n] = torch.from_numpy(w)
    pl = ozaki.plan(n, beta, beta)
    eb = ozaki.encode(wd, n, n, "b", pl)
    ea = ozaki.encode(wd, n, n, "a", pl)
    res = ozaki.ResidueBuffer(n, n, pl.nmod, "cuda")
    w2 = lp_empty(n, dtype=dtype)
    ozaki.gemm_residues(ea, eb, pl, res, lower_only=True)
    ozaki.decode(res, ea, eb, pl, w2, hermitian=True)
    ea2 = ozaki.encode(w2, n, n, "a", pl)
    w3 = lp_empty(n, dtype=dtype)
    ozaki.gemm_residues(ea2, eb, pl, res, lower_only=True)
    ozaki.decode(res, ea2, eb, pl, w3, hermitian="skew")
    wc = w.astype(np.complex128)
    g2, g3 = w2[:, :n].cpu().numpy(), w3[:, :n].cpu().numpy()
    tol = 1e-6 if dtype == torch.complex64 else 1e-14
    assert np.linalg.norm(g2 - wc @ wc) <= tol * np.linalg.norm(wc @ wc)
    assert np.linalg.norm(g3 - g2.astype(np.complex128) @ wc) <= tol * np.linalg.norm(wc @ wc @ wc)
    up = np.zeros((n, n), bool)  # strictly-upper 128-tiles: mirrored
    for i in range(n):
        up[i, (i // 128 + 1) * 128:] = True
    assert np.array_equal(g2[up], g2.conj().T[up])
    assert np.array_equal(g3[up], -g3.conj().T[up])


def test_oz_encode_dual_matches_two_encodes():
    """sr_oz_encode_dual writes exactly the residues (and exponents) of the two
    separate encodes of Q^H (A role) and Q (B role)."""
    rng = np.random.default_rng(5)
    n = 300
    q = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    q[:, 7] *= 1e-9  # a small column: its own exponent
    qd = ZPlanar.from_any(q)
    pl = ozaki.plan(n, ozaki.HP_BETA, ozaki.HP_BETA)
    ea = ozaki.encode(qd, n, n, "a", pl, conj_t=True)
    eb = ozaki.encode(qd, n, n, "b", pl)
    da = ozaki.Encoded(n, n, 2, pl.beta_a, pl.nmod, "cuda")
    db = ozaki.Encoded(n, n, 3, pl.beta_b, pl.nmod, "cuda")
    ozaki.encode_dual(qd, n, n, pl, da, db)
    assert torch.equal(ea.buf, da.buf) and torch.equal(eb.buf, db.buf)
    assert torch.equal(ea.exps, da.exps) and torch.equal(eb.exps, db.exps)


# ---- Gaussian-CRT products (two real products per modulus) -------------------

GMODS = [241, 233, 229, 221]


@pytest.mark.parametrize("M,N,K,b_planes,a_swap,herm", [
    (128, 128, 64, 2, 0, 0), (200, 130, 100, 2, 1, 0), (256, 384, 512, 1, 0, 0), (77, 300, 1000, 1, 1, 0),
    (300, 300, 129, 2, 1, 1), (129, 129, 70, 2, 0, -1), (384, 384, 256, 2, 0, 1), (200, 300, 96, 2, 2, 0),
    (256, 256, 128, 2, 3, 0), (300, 300, 64, 2, 2, 1)])
def test_oz_gemm_gauss_bit_exact(M, N, K, b_planes, a_swap, herm):
    rng = np.random.default_rng(M * 3 + N + K + herm)
    kp = ozaki.kpitch(K)
    a = np.zeros((len(GMODS), 2, M, kp), np.int8)
    b = np.zeros((len(GMODS), b_planes, N, kp), np.int8)
    for l, p in enumerate(GMODS):
        a[l, :, :, :K] = sym_residues(rng, (2, M, K), p)
        b[l, :, :, :K] = sym_residues(rng, (b_planes, N, K), p)
    ad, bd = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    pitch = ozaki.kpitch(N)
    out = torch.zeros((len(GMODS), 2, M, pitch), dtype=torch.int8, device="cuda")
    mods = np.array(GMODS, np.int32)
    rc = _lib.call("sr_oz_gemm_i8_gauss", M, N, K, len(GMODS), mods.ctypes.data, ad.data_ptr(), a_swap, kp,
                   bd.data_ptr(), b_planes, kp, out.data_ptr(), pitch, herm, 0, torch.cuda.current_stream().cuda_stream)
    assert rc is None or rc == 0
    got = out.cpu().numpy()[:, :, :, :N].astype(np.int64)
    for l, p in enumerate(GMODS):
        sa, sb = a_swap & 1, (a_swap >> 1) & 1  # bit 1: B planes swapped
        c = [a[l, g ^ sa].astype(np.int64) @ b[l, (g ^ sb) if b_planes == 2 else 0].astype(np.int64).T
             for g in (0, 1)]
        assert np.array_equal(got[l, 0], sym_mod(c[0], p)), (l, p)
        if herm:
            assert np.array_equal(got[l, 1], sym_mod(herm * c[0].T, p)), (l, p)
        else:
            assert np.array_equal(got[l, 1], sym_mod(c[1], p)), (l, p)


def oz_product_gauss(x, y, trans=False, alpha=1.0, shift=0.0, beta=ozaki.HP_BETA):
    xm, ym = ZPlanar.from_any(x), ZPlanar.from_any(y)
    K = x.shape[0] if trans else x.shape[1]
    M = x.shape[1] if trans else x.shape[0]
    N = y.shape[1]
    pl = ozaki.gauss_plan(K, beta, beta)
    ea = ozaki.encode(xm, x.shape[0], x.shape[1], "a", pl, conj_t=trans)
    eb = ozaki.encode(ym, y.shape[0], y.shape[1], "b", pl)
    res = ozaki.ResidueBuffer(M, N, pl.nmod, "cuda")
    ozaki.gemm_residues(ea, eb, pl, res)
    out = ZPlanar.empty(M, N)
    ozaki.decode(res, ea, eb, pl, out, alpha=alpha, shift=shift)
    return out.to_numpy()


@pytest.mark.parametrize("M,N,K", [(1, 1, 1), (64, 48, 40), (200, 130, 257), (256, 256, 256)])
@pytest.mark.parametrize("trans", [False, True])
@pytest.mark.parametrize("b_real", [False, True])
def test_oz_gauss_fp64_product_beats_blas(M, N, K, trans, b_real):
    rng = np.random.default_rng(M * 5 + N + K)
    x = rng.standard_normal((K, M) if trans else (M, K)) + 1j * rng.standard_normal((K, M) if trans else (M, K))
    y = rng.standard_normal((K, N))
    if not b_real:
        y = y + 1j * rng.standard_normal((K, N))
    xo = x.conj().T if trans else x
    exact, _ = dd_exact(xo, y)
    got = oz_product_gauss(x, y, trans=trans)
    blas = xo @ y
    e_oz = np.linalg.norm(got - exact)
    e_blas = np.linalg.norm(blas - exact)
    scale = np.linalg.norm(exact)
    assert e_oz <= max(2 * e_blas, 4 * 2.0 ** -53 * scale), (e_oz / scale, e_blas / scale)


@pytest.mark.parametrize("n", [200, 300])
def test_oz_gauss_gram_from_one_encoding(n):
    """Y = Q^H Q - I from ONE encoding of Q (its B operand, read with swapped
    planes as the A operand of Q^H) and one real product per modulus (herm)."""
    rng = np.random.default_rng(11)
    q, _ = np.linalg.qr(rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)))
    _, o = dd_exact(q.conj().T, q)
    exact = (o[0] - np.eye(n)) + o[1] + 1j * (o[2] + o[3])
    pl = ozaki.gauss_plan(n, ozaki.HP_BETA, ozaki.HP_BETA)
    eb = ozaki.encode(ZPlanar.from_any(q), n, n, "b", pl)
    res = ozaki.ResidueBuffer(n, n, pl.nmod, "cuda")
    ozaki.gemm_residues(ozaki.conj_view(eb), eb, pl, res, lower_only=True)
    out = ZPlanar.empty(n, n)
    ozaki.decode(res, ozaki.conj_view(eb), eb, pl, out, shift=-1.0, hermitian=True)
    got = out.to_numpy()
    blas = q.conj().T @ q - np.eye(n)
    assert np.array_equal(got, got.conj().T)
    assert np.linalg.norm(got - exact) <= np.linalg.norm(blas - exact)
    # the same product from the explicit conj-transposed encoding, no Hermitian shortcut
    assert np.array_equal(got, oz_product_gauss(q, q, trans=True, shift=-1.0))


@pytest.mark.parametrize("n", [300, 515])
def test_oz_gauss_lp_structured_products(n):
    """complex64 W = L - L^H: W^2 (Hermitian, one real product per modulus,
    exactly Hermitian) and W^3 = W^2 W (a full product: row i of W^2 and
    column i of W are scaled differently, so the integer product is not
    skew-Hermitian and the transpose shortcut does not apply); lp accuracy."""
    rng = np.random.default_rng(n + 1)
    l = np.tril(rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)), -1) * 1e-3
    w = (l - l.conj().T).astype(np.complex64)
    wd = lp_empty(n)
    wd[:, :n] = torch.from_numpy(w)
    pl = ozaki.gauss_plan(n, ozaki.LP_BETA, ozaki.LP_BETA)
    eb = ozaki.encode(wd, n, n, "b", pl)
    ea = ozaki.encode(wd, n, n, "a", pl)
    res = ozaki.ResidueBuffer(n, n, pl.nmod, "cuda")
    w2 = lp_empty(n)
    ozaki.gemm_residues(ea, eb, pl, res, lower_only=True)
    ozaki.decode(res, ea, eb, pl, w2, hermitian=True)
    ea2 = ozaki.encode(w2, n, n, "a", pl)
    w3 = lp_empty(n)
    ozaki.gemm_residues(ea2, eb, pl, res, lower_only="skew")
    ozaki.decode(res, ea2, eb, pl, w3, hermitian="skew")
    wc = w.astype(np.complex128)
    g2, g3 = w2[:, :n].cpu().numpy(), w3[:, :n].cpu().numpy()
    assert np.linalg.norm(g2 - wc @ wc) <= 1e-6 * np.linalg.norm(wc @ wc)
    assert np.linalg.norm(g3 - g2.astype(np.complex128) @ wc) <= 1e-6 * np.linalg.norm(wc @ wc @ wc)
    assert np.array_equal(g2, g2.conj().T)
