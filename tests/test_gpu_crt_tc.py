"""Tensor-core CRT decode (csrc/ozaki.cu: decode_tc_kernel) against the SIMT
decode (decode_kernel) on the same residues.

Both form the same exact integer chunk sums S_j and run the same CRT finish,
so the bar is bit-identical outputs (integer work), on real products (encode
+ modular GEMM of random operands) and on uniformly random residues, for
every Gaussian output kind the FP64 mode uses: planar FP64 (plain, alpha /
shift / diagonal offset, + X), Hermitian lower-tile decodes, complex64.
"""
import numpy as np
import pytest
import torch

from paper_2203_10879_b200 import ZPlanar, _lib, ozaki
from paper_2203_10879_b200.matrix import lp_empty

pytestmark = pytest.mark.gpu


def _both(fn):
    """fn() with the SIMT decode, then with the tensor-core decode."""
    lib = _lib.load()
    old = lib.sr_oz_config(0, -1)
    outs = []
    try:
        for mode in (0, 1):
            lib.sr_oz_config(0, mode)
            outs.append(fn())
            torch.cuda.synchronize()
    finally:
        lib.sr_oz_config(0, old)
    return outs


def _planes_equal(a, b):
    if isinstance(a, torch.Tensor):
        return torch.equal(a, b)
    return torch.equal(a.re, b.re) and torch.equal(a.im, b.im)


def _rand_zp(n, m, seed, scale=1.0):
    g = torch.Generator().manual_seed(seed)
    x = torch.complex(torch.randn(n, m, generator=g, dtype=torch.float64),
                      torch.randn(n, m, generator=g, dtype=torch.float64)) * scale
    return ZPlanar.from_any(x.cuda())


@pytest.mark.parametrize("n", [128, 300, 517])
@pytest.mark.parametrize("variant", ["plain", "add", "shift"])
def test_decode_tc_hp_product_bit_identical(n, variant):
    a, b = _rand_zp(n, n, n), _rand_zp(n, n, n + 1)
    pl = ozaki.plan(n, ozaki.HP_BETA, ozaki.HP_BETA, gauss=True)
    ea = ozaki.encode(a, n, n, "a", pl, conj_t=True)
    eb = ozaki.encode(b, n, n, "b", pl)
    res = ozaki.ResidueBuffer(n, n, pl.nmod, "cuda")
    ozaki.gemm_residues(ea, eb, pl, res)
    x = _rand_zp(n, n, 7)

    def run():
        out = ZPlanar.empty(n)
        if variant == "plain":
            ozaki.decode(res, ea, eb, pl, out)
        elif variant == "add":
            ozaki.decode(res, ea, eb, pl, out, alpha=0.5, add=x)
        else:
            ozaki.decode(res, ea, eb, pl, out, alpha=-1.0, shift=-1.0)
        return out

    simt, tc = _both(run)
    assert _planes_equal(simt, tc)
    assert torch.isfinite(tc.re[:, :n]).all()


@pytest.mark.parametrize("n", [200, 384])
def test_decode_tc_hermitian_bit_identical(n):
    q = _rand_zp(n, n, 11)
    pl = ozaki.plan(n, ozaki.HP_BETA_Q, ozaki.HP_BETA_Q, gauss=True)
    eb = ozaki.encode(q, n, n, "b", pl)
    ea = ozaki.conj_view(eb)
    res = ozaki.ResidueBuffer(n, n, pl.nmod, "cuda")
    ozaki.gemm_residues(ea, eb, pl, res, lower_only=True)

    def run():
        out = ZPlanar.empty(n)
        ozaki.decode(res, ea, eb, pl, out, shift=-1.0, hermitian=True)
        return out

    simt, tc = _both(run)
    assert _planes_equal(simt, tc)


@pytest.mark.parametrize("n", [130, 260])
def test_decode_lp_bit_identical(n):
    """lp (2 kept chunks) stays on the SIMT decode; both settings must agree."""
    g = torch.Generator().manual_seed(n)
    a, b = lp_empty(n), lp_empty(n)
    a[:, :n] = torch.randn(n, n, generator=g, dtype=torch.complex64).cuda()
    b[:, :n] = torch.randn(n, n, generator=g, dtype=torch.complex64).cuda()
    pl = ozaki.plan(n, ozaki.LP_BETA, ozaki.LP_BETA, gauss=True)
    ea = ozaki.encode(a, n, n, "a", pl)
    eb = ozaki.encode(b, n, n, "b", pl)
    res = ozaki.ResidueBuffer(n, n, pl.nmod, "cuda")
    ozaki.gemm_residues(ea, eb, pl, res)

    def run():
        out = lp_empty(n)
        out.zero_()
        ozaki.decode(res, ea, eb, pl, out)
        return out

    simt, tc = _both(run)
    assert torch.equal(simt, tc)


@pytest.mark.parametrize("K,beta,out_bits", [(8192, 58, 53), (1024, 58, 53), (8192, 24, 24), (64, 58, 53),
                                             (8192, 40, 53)])
def test_decode_tc_random_residues_bit_identical(K, beta, out_bits):
    """Uniformly random residues (C' anywhere in (-P/2, P/2)) for the plans the
    refinement uses (nmod up to 19, 2 to 4 kept chunks)."""
    pl = ozaki.plan(K, beta, beta, gauss=True)
    nchunk = pl.decode_chunks(out_bits)
    assert 2 <= nchunk <= 4 and pl.nmod <= 32
    M, N = 257, 300
    rng = np.random.default_rng(K + beta)
    res = ozaki.ResidueBuffer(M, N, pl.nmod, "cuda")
    host = np.zeros((pl.nmod, 2, M, res.pitch), np.int8)
    for l, p in enumerate(pl.moduli):
        host[l, :, :, :N] = rng.integers(-(p // 2), (p + 1) // 2, size=(2, M, N))
    res.buf.copy_(torch.from_numpy(host.reshape(-1)))

    class E:  # encodings: only the exponents and betas are read by the decode
        pass

    ea, eb = E(), E()
    ea.exps = torch.full((M,), 3, dtype=torch.int32, device="cuda")
    eb.exps = torch.tensor(rng.integers(-4, 4, size=N), dtype=torch.int32, device="cuda")
    ea.beta, eb.beta = pl.beta_a, pl.beta_b

    def run():
        if out_bits == 24:
            out = torch.zeros((M, N), dtype=torch.complex64, device="cuda")
        else:
            out = ZPlanar.empty(M, N)
        ozaki.decode(res, ea, eb, pl, out)
        return out

    simt, tc = _both(run)
    assert _planes_equal(simt, tc)


def test_config_query_and_unknown_key():
    lib = _lib.load()
    cur = lib.sr_oz_config(0, -1)
    assert cur in (0, 1)
    assert lib.sr_oz_config(99, 1) == -1
    assert lib.sr_oz_config(0, -1) == cur


def _exact_gauss_decode(host, pl, rho, sigma, M, N, alpha=1.0):
    """Exact Gaussian CRT reconstruction (Python integers / Fractions), correctly
    rounded to binary64: the reference the decode is held to."""
    from fractions import Fraction
    P = pl.P
    ws = []
    for p in pl.moduli:
        m = P // p
        ws.append((m * pow(m % p, -1, p)) % P)
    re = np.zeros((M, N))
    im = np.zeros((M, N))
    for i in range(M):
        for j in range(N):
            cr = ci = 0
            for l, p in enumerate(pl.moduli):
                a, b = int(host[l, 0, i, j]), int(host[l, 1, i, j])
                io = ozaki.sqrt_minus_one(p)
                cr += ((a + b) * pow(2, -1, p) % p) * ws[l]
                ci += ((a - b) * pow(2 * io, -1, p) % p) * ws[l]
            cr, ci = cr % P, ci % P
            cr = cr - P if cr > P // 2 else cr
            ci = ci - P if ci > P // 2 else ci
            sc = Fraction(1, 2 ** int(rho[i] + sigma[j]))
            re[i, j] = float(Fraction(cr) * sc * Fraction(alpha))
            im[i, j] = float(Fraction(ci) * sc * Fraction(alpha))
    return re, im


@pytest.mark.parametrize("tc", [0, 1])
def test_gauss_decode_correctly_rounded(tc):
    """Both Gaussian decodes (SIMT, tensor core) against the exact CRT value of
    random residues (C' anywhere in (-P/2, P/2)): correctly rounded except for
    a rare double rounding, never more than 1 ulp off."""
    K, beta = 8192, 58
    pl = ozaki.plan(K, beta, beta, gauss=True)
    M, N = 40, 70
    rng = np.random.default_rng(5)
    res = ozaki.ResidueBuffer(M, N, pl.nmod, "cuda")
    host = np.zeros((pl.nmod, 2, M, res.pitch), np.int8)
    for l, p in enumerate(pl.moduli):
        host[l, :, :, :N] = rng.integers(-(p // 2), (p + 1) // 2, size=(2, M, N))
    res.buf.copy_(torch.from_numpy(host.reshape(-1)))

    class E:
        pass

    ea, eb = E(), E()
    ea_e = rng.integers(-3, 3, size=M)
    eb_e = rng.integers(-3, 3, size=N)
    ea.exps = torch.tensor(ea_e, dtype=torch.int32, device="cuda")
    eb.exps = torch.tensor(eb_e, dtype=torch.int32, device="cuda")
    ea.beta, eb.beta = pl.beta_a, pl.beta_b
    lib = _lib.load()
    old = lib.sr_oz_config(0, tc)
    try:
        out = ZPlanar.empty(M, N)
        ozaki.decode(res, ea, eb, pl, out, alpha=-0.5)
        torch.cuda.synchronize()
    finally:
        lib.sr_oz_config(0, old)
    rho = pl.beta_a - ea_e
    sigma = pl.beta_b - eb_e
    ere, eim = _exact_gauss_decode(host, pl, rho, sigma, M, N, alpha=-0.5)
    for got, exact in ((out.re.cpu().numpy(), ere), (out.im.cpu().numpy(), eim)):
        ulp = np.spacing(np.abs(exact))
        err = np.abs(got - exact) / ulp
        assert err.max() <= 1.0, err.max()
        assert np.mean(got == exact) >= 0.999, np.mean(got == exact)


@pytest.fixture(autouse=False)
def fit_all_sizes(monkeypatch):
    monkeypatch.setattr(ozaki, "FIT_MIN_K", 0)


def _product(a, b, n, pl, fit):
    ea = ozaki.encode(a, n, n, "a", pl, conj_t=True)
    eb = ozaki.encode(b, n, n, "b", pl)
    use = ozaki.fit_plan(pl, ea, eb) if fit else pl
    res = ozaki.ResidueBuffer(n, n, pl.nmod, "cuda")
    ozaki.gemm_residues(ea, eb, use, res)
    out = ZPlanar.empty(n)
    ozaki.decode(res, ea, eb, use, out)
    torch.cuda.synchronize()
    return out, use.nmod


@pytest.mark.parametrize("kind", ["unitary", "gaussian", "flat", "graded"])
@pytest.mark.parametrize("n", [256, 1024])
def test_fit_plan_is_exact(kind, n, fit_all_sizes):
    """fit_plan keeps only the moduli the Cauchy-Schwarz bound of the integer-
    scaled operands requires; the CRT value is then the same integer, so the
    decoded product agrees with the worst-case plan's to the decode's chunk
    truncation — including for 'flat' operands (every entry of equal
    magnitude, the bound's worst case) and rows graded by 2^+-20."""
    g = torch.Generator().manual_seed(n + len(kind))
    if kind == "unitary":
        x = torch.complex(torch.randn(n, n, generator=g, dtype=torch.float64),
                          torch.randn(n, n, generator=g, dtype=torch.float64))
        a = torch.linalg.qr(x)[0]
        b = a
    elif kind == "gaussian":
        a = torch.complex(torch.randn(n, n, generator=g, dtype=torch.float64),
                          torch.randn(n, n, generator=g, dtype=torch.float64))
        b = torch.complex(torch.randn(n, n, generator=g, dtype=torch.float64),
                          torch.randn(n, n, generator=g, dtype=torch.float64))
    elif kind == "flat":
        a = torch.polar(torch.ones(n, n, dtype=torch.float64), torch.rand(n, n, generator=g, dtype=torch.float64) * 6.283)
        b = torch.polar(torch.ones(n, n, dtype=torch.float64), torch.rand(n, n, generator=g, dtype=torch.float64) * 6.283)
    else:
        a = torch.complex(torch.randn(n, n, generator=g, dtype=torch.float64),
                          torch.randn(n, n, generator=g, dtype=torch.float64))
        a = a * torch.exp2(torch.randint(-20, 20, (n, 1), generator=g).double())
        b = a.conj().T.contiguous()
    A, B = ZPlanar.from_any(a.cuda()), ZPlanar.from_any(b.cuda())
    pl = ozaki.plan(n, ozaki.HP_BETA, ozaki.HP_BETA, gauss=True)
    full, m_full = _product(A, B, n, pl, fit=False)
    fit, m_fit = _product(A, B, n, pl, fit=True)
    assert m_fit <= m_full
    if kind == "unitary":
        assert m_fit < m_full  # ||q_i|| = 1: at least one modulus less
    # the same CRT integer C'; the decodes keep the top chunks of different
    # moduli products, so they agree to far below the operands' own 2^-58
    # truncation (relative to |a_i|_inf |b_j|_inf): exact CRT, no wraparound
    fa = full.re[:, :n].cpu().numpy() + 1j * full.im[:, :n].cpu().numpy()
    fb = fit.re[:, :n].cpu().numpy() + 1j * fit.im[:, :n].cpu().numpy()
    an, bn = a.numpy(), b.numpy()
    scale = np.abs(an.conj().T).max(axis=1)[:, None] * np.abs(bn).max(axis=0)[None, :]
    assert np.max(np.abs(fa - fb) / scale) <= 2.0 ** -70
    ref = an.conj().T @ bn
    assert np.max(np.abs(fb - ref) / scale) <= 2.0 ** -40
