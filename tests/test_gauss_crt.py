"""CPU checks of the Gaussian-CRT plan (ozaki.OzPlan(gauss=True)).

For moduli p with a square root iota of -1, x + iy -> (x + iota y, x - iota y)
is a ring isomorphism Z[i]/p -> Z/p x Z/p, so a complex integer product mod p
is two real products.  These tests model the device pipeline with exact
Python integers — encode to (phi+, phi-), multiply per plane, recombine with
the plan's CRT table exactly as csrc/ozaki.cu's decode_kernel<..., G> reads it
— and require the exact complex integer product back.  Integer work: the bar
is equality."""
import math

import numpy as np
import pytest

from paper_2203_10879_b200 import ozaki


def _sym(x, p):
    r = x % p
    return r - p if r > (p + 1) // 2 - 1 else r


def _table_weights(pl):
    """(w_re, w_im, P) as integers, rebuilt from the float chunks of pl.table."""
    M = ozaki.MAXCHUNK
    t = pl.table
    n = pl.nmod
    offs = [int(o) for o in t[n * M + M:n * M + 2 * M]]

    def whole(ch):
        return sum(int(c) << offs[j] for j, c in enumerate(ch[:pl.nchunk]))
    w_re = [whole(t[l * M:(l + 1) * M]) for l in range(n)]
    P = whole(t[n * M:n * M + M])
    base = n * M + 2 * M + 1
    w_im = [whole(t[base + l * M:base + (l + 1) * M]) for l in range(n)]
    return w_re, w_im, P


def test_gauss_moduli_are_coprime_with_sqrt_minus_one():
    mods = ozaki.GAUSS_MODULI
    for i, p in enumerate(mods):
        assert p % 2 == 1 and p <= 256
        io = ozaki.sqrt_minus_one(p)
        assert (io * io + 1) % p == 0
        for q in mods[i + 1:]:
            assert math.gcd(p, q) == 1


@pytest.mark.parametrize("beta,K", [(58, 8192), (24, 8192), (58, 256), (30, 7)])
def test_gauss_plan_covers_the_product_bound(beta, K):
    pl = ozaki.gauss_plan(K, beta, beta)
    assert pl.P >= 2 * 2 * K * 2 ** (2 * beta)
    assert pl.nmod * 240 * 2 ** ozaki.CHUNK_BITS < 2 ** 53  # decode chunk sums stay exact


@pytest.mark.parametrize("seed,M,K,N,beta", [(0, 3, 5, 4, 20), (1, 6, 9, 2, 58), (2, 4, 16, 4, 40)])
@pytest.mark.parametrize("conj_a", [False, True])
def test_gauss_crt_reconstructs_complex_products(seed, M, K, N, beta, conj_a):
    rng = np.random.default_rng(seed)
    pl = ozaki.gauss_plan(K, beta, beta)
    lim = 2 ** beta

    def rand(rows, cols):  # complex integers as (re, im) pairs below 2^beta
        return [[(int(rng.integers(-lim, lim)), int(rng.integers(-lim, lim))) for _ in range(cols)]
                for _ in range(rows)]
    A = rand(M, K)
    B = rand(K, N)
    if conj_a:  # the A operand of X^H from X's own phi planes with the planes swapped
        X = [[A[i][k] for i in range(M)] for k in range(K)]  # K x M, A = X^H below
        A = [[(X[k][i][0], -X[k][i][1]) for k in range(K)] for i in range(M)]
    w_re, w_im, P = _table_weights(pl)
    assert P == pl.P
    for i in range(M):
        for j in range(N):
            cre = sum(A[i][k][0] * B[k][j][0] - A[i][k][1] * B[k][j][1] for k in range(K))
            cim = sum(A[i][k][0] * B[k][j][1] + A[i][k][1] * B[k][j][0] for k in range(K))
            sre = sim = 0
            for l, p in enumerate(pl.moduli):
                io = ozaki.sqrt_minus_one(p)
                if conj_a:
                    # phi+(conj z) = phi-(z): X's planes read swapped
                    ap = [_sym(X[k][i][0] - io * X[k][i][1], p) for k in range(K)]
                    am = [_sym(X[k][i][0] + io * X[k][i][1], p) for k in range(K)]
                else:
                    ap = [_sym(A[i][k][0] + io * A[i][k][1], p) for k in range(K)]
                    am = [_sym(A[i][k][0] - io * A[i][k][1], p) for k in range(K)]
                bp = [_sym(B[k][j][0] + io * B[k][j][1], p) for k in range(K)]
                bm = [_sym(B[k][j][0] - io * B[k][j][1], p) for k in range(K)]
                cp = _sym(sum(x * y for x, y in zip(ap, bp)), p)
                cm = _sym(sum(x * y for x, y in zip(am, bm)), p)
                sre += (cp + cm) * w_re[l]
                sim += (cp - cm) * w_im[l]
            assert _sym(sre, P) == cre
            assert _sym(sim, P) == cim


def test_gauss_hermitian_planes_are_transposes():
    """C = X^H X Hermitian: phi-(C) = phi+(C)^T, so one real product suffices."""
    rng = np.random.default_rng(4)
    n, K, p = 5, 7, 241
    io = ozaki.sqrt_minus_one(p)
    X = rng.integers(-50, 50, size=(K, n)) + 1j * rng.integers(-50, 50, size=(K, n))
    C = X.conj().T @ X
    cp = np.vectorize(lambda z: _sym(int(z.real) + io * int(z.imag), p))(C)
    cm = np.vectorize(lambda z: _sym(int(z.real) - io * int(z.imag), p))(C)
    assert np.array_equal(cm, cp.T)
    W = X[:n, :n] - X[:n, :n].conj().T  # skew-Hermitian: phi-(W) = -phi+(W)^T
    wp = np.vectorize(lambda z: _sym(int(z.real) + io * int(z.imag), p))(W)
    wm = np.vectorize(lambda z: _sym(int(z.real) - io * int(z.imag), p))(W)
    assert np.array_equal(wm, np.vectorize(lambda v: _sym(-v, p))(wp.T))
