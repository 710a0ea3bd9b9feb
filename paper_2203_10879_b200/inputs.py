"""Seeded synthetic inputs for the BASELINE.json configs.

Not part of the refinement path: these build the matrices A and the
starting candidates Q̂ the benchmark and the parity tests feed to
`refine_template`.  RNG convention is the reference's
(`/root/reference/pkg/src/ddschur/generators.py:84-85`): a Philox
generator, real part drawn before the imaginary part, each one full
C-order (n, n) `standard_normal` block.

Q̂ is LAPACK's complex Schur vector matrix (`scipy.linalg.schur`,
cgees/zgees, LAPACK eigenvalue order).  It is computed once per
(config, n, seed) and cached as `.npy` under $SR_DATA_DIR (default /tmp/sr_data, outside the
repo: the n = 8192 matrix alone is 512 MiB) because cgees at n = 8192 takes
minutes.  The cache only shortens setup; no timed region depends on it.
"""
import os

import numpy as np

_DATA = os.environ.get("SR_DATA_DIR", "/tmp/sr_data")


def _rng(seed):
    return np.random.Generator(np.random.Philox(int(seed)))


def gaussian_complex(n, seed=0, rng=None):
    """A with re, im each N(0, 1/2) (configs 1, 2, 5)."""
    rng = _rng(seed) if rng is None else rng
    re = rng.standard_normal((n, n))
    im = rng.standard_normal((n, n))
    return (re + 1j * im) * np.sqrt(0.5)


def gaussian_real(n, seed=0):
    """A real N(0, 1) (config 3)."""
    return _rng(seed).standard_normal((n, n))


def haar_unitary(n, rng):
    """QR of a complex Gaussian with the diagonal phase fixed (Haar)."""
    z = (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))) * np.sqrt(0.5)
    q, r = np.linalg.qr(z)
    d = np.diagonal(r)
    return q * (d / np.abs(d))[None, :]


def config4_matrix(n=1024, seed=0, strict_scale=1.0):
    """A = U T0 U^H, T0 = triu(N(0,1/2)-complex, 1) * strict_scale + diag(lambda_k),
    lambda_k = exp(2 pi i k / n) (1 + k / n), k = 0..n-1 (BASELINE config 4).
    strict_scale = 1/sqrt(n) gives the documented well-conditioned variant."""
    rng = _rng(seed)
    u = haar_unitary(n, rng)
    s = (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))) * np.sqrt(0.5)
    k = np.arange(n)
    lam = np.exp(2j * np.pi * k / n) * (1.0 + k / n)
    t0 = np.triu(s, 1) * strict_scale + np.diag(lam)
    return (u @ t0) @ u.conj().T


def config5_pair(n=512, seed=0):
    """A0, A1 complex Gaussian from one Philox stream (config 5)."""
    rng = _rng(seed)
    a0 = gaussian_complex(n, rng=rng)
    a1 = gaussian_complex(n, rng=rng)
    return a0, a1


def schur_vectors(a, dtype=np.complex64):
    """Complex Schur vectors of a cast to dtype (LAPACK cgees / zgees)."""
    import scipy.linalg

    x = np.asarray(a).astype(dtype)
    _, z = scipy.linalg.schur(x, output="complex")
    return z


def cached_qhat(tag, a, dtype=np.complex64):
    """schur_vectors(a) cached under $SR_DATA_DIR/qhat_<tag>.npy."""
    os.makedirs(_DATA, exist_ok=True)
    path = os.path.join(_DATA, "qhat_%s.npy" % tag)
    if os.path.exists(path):
        z = np.load(path)
        if z.shape == a.shape:
            return z
    z = schur_vectors(a, dtype)
    tmp = path + ".tmp.npy"
    np.save(tmp, z)
    os.replace(tmp, path)
    return z


def config_inputs(cfg, n=None, seed=0):
    """(A, Q̂) for BASELINE config 1, 2, 3 or 4 (complex Q̂ as complex128)."""
    if cfg in (1, 2):
        n = n or (256 if cfg == 1 else 2048)
        a = gaussian_complex(n, seed)
        q = cached_qhat("c%d_n%d_s%d" % (cfg, n, seed), a)
    elif cfg == 3:
        n = n or 8192
        a = gaussian_real(n, seed)
        q = cached_qhat("c3_n%d_s%d" % (n, seed), a)
    elif cfg == 4:
        n = n or 1024
        a = config4_matrix(n, seed)
        q = cached_qhat("c4_n%d_s%d" % (n, seed), a, dtype=np.complex128)
    else:
        raise ValueError("config must be 1..4 (config 5 is config5_pair)")
    return a, q.astype(np.complex128)
