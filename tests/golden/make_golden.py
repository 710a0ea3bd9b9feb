"""Generate the committed golden fixtures from the REAL reference.

Run in the build container only (needs /root/reference, which never
exists on the GPU box):

    python tests/golden/make_golden.py

The reference is copied to /tmp first so numba's on-disk cache never
writes into the read-only reference tree.  Every fixture
records the reference call that produced it.  The fixtures are the pins
for `oracle/` (tests/test_oracle.py) and the targets of the GPU parity
tests (tests/test_gpu_parity.py).
"""
import json
import os
import shutil
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
REF_SRC = "/root/reference/pkg/src"
TMP_REF = "/tmp/ddschur_ref_copy"


def import_reference():
    if not os.path.isdir(TMP_REF):
        shutil.copytree(REF_SRC, TMP_REF)
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_golden")
    sys.path.insert(0, TMP_REF)
    sys.path.insert(0, REPO)
    import ddschur  # noqa: F401
    return ddschur


def random_upper(rng, n, diag_sep=1.0, scale=1.0):
    t = scale * (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)))
    t = np.triu(t)
    spread = np.cumsum(diag_sep + rng.uniform(0.0, 1.0, size=n))
    phases = np.exp(1j * rng.uniform(0.0, 2 * np.pi, size=n))
    t[np.arange(n), np.arange(n)] = spread * phases
    return t


def gen_trisolve(ref):
    """solve_block on seeded (T, E); clip off / on; n_min 2 and 4."""
    from ddschur.trisolve import TriEqProblem, solve_block
    out = {}
    cases = []
    k = 0
    for n in (2, 3, 4, 5, 7, 8, 13, 16, 31, 32, 33, 64, 100):
        for clip in (None, 0.05):
            for n_min in (2, 4):
                rng = np.random.Generator(np.random.Philox(1000 + k))
                t = random_upper(rng, n)
                e = np.tril(rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)), -1)
                e *= 0.1
                sol = solve_block(TriEqProblem(t=t, e=e, clip_threshold=clip), n_min=n_min)
                out["t_%d" % k] = t
                out["e_%d" % k] = e
                out["l_%d" % k] = sol.l
                cases.append(dict(k=k, n=n, clip=clip, n_min=n_min, clipped=int(sol.clipped_count)))
                k += 1
    np.savez_compressed(os.path.join(HERE, "trisolve_ref.npz"), **out)
    with open(os.path.join(HERE, "trisolve_ref.json"), "w") as f:
        json.dump(dict(source="ddschur.trisolve.solve_block (trisolve.py:243-262)", cases=cases), f, indent=1)


def gen_ddgemm(ref):
    """matmul_hp (numba gemm_hp, panel 32) on seeded normalised dd inputs."""
    from ddschur.ddmatrix import DDMatrix
    from ddschur.matmul import matmul_hp
    out = {}
    meta = []
    for k, (m, kk, n) in enumerate(((5, 7, 3), (16, 16, 16), (33, 70, 20), (64, 64, 64))):
        rng = np.random.Generator(np.random.Philox(2000 + k))

        def dd(shape):
            hi = rng.standard_normal(shape) + 0j + 1j * rng.standard_normal(shape)
            lo = (rng.standard_normal(shape) + 1j * rng.standard_normal(shape)) * 2.0 ** -60
            rh, rl = hi.real + lo.real, None
            # normalise each (hi, lo) pair with an exact two_sum
            def norm(h, l_):
                s = h + l_
                bb = s - h
                e = (h - (s - bb)) + (l_ - bb)
                return s, e
            rh, rl = norm(hi.real, lo.real)
            ih, il = norm(hi.imag, lo.imag)
            return DDMatrix(rh, rl, ih, il)
        a = dd((m, kk))
        b = dd((kk, n))
        c = matmul_hp(a, b)
        for name, mat in (("a", a), ("b", b), ("c", c)):
            for cell, arr in zip(("rh", "rl", "ih", "il"), mat.cells()):
                out["%s%s_%d" % (name, cell, k)] = np.ascontiguousarray(arr)
        meta.append(dict(k=k, m=m, k_dim=kk, n=n))
    np.savez_compressed(os.path.join(HERE, "ddgemm_ref.npz"), **out)
    with open(os.path.join(HERE, "ddgemm_ref.json"), "w") as f:
        json.dump(dict(source="ddschur.matmul.matmul_hp (numba gemm_hp, panel 32)", cases=meta), f, indent=1)


def make_instance(ref, rng, n, strict=0.5):
    """A = U T U^H with separated eigenvalues, as in test_refine.py's
    construction (diag spacing >= 0.7); candidate = U * cubic exp slice."""
    from ddschur.ddmatrix import DDMatrix
    from ddschur.matmul import matmul_hp
    from ddschur.orthogonal import qr_retract
    t = np.triu(strict * (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))), 1)
    diag = np.arange(n) + 0.7 * rng.random(n) + 1j * rng.uniform(-1.0, 1.0, n)
    t = t + np.diag(diag)
    m = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    u = qr_retract(DDMatrix.from_lp(m))
    a = matmul_hp(matmul_hp(u, DDMatrix.from_lp(t)), u, trans_b=True)
    return a, u


def gen_refine_dd(ref):
    """refine_template in the reference's native dd mode on small seeded
    instances: A = U T U^H, Q̂ = U * (I + K + K^2/2 + K^3/6), ||K|| = eps."""
    from ddschur.ddmatrix import DDMatrix
    from ddschur.matmul import matmul_hp
    from ddschur.refine import RefineConfig, refine_template, verify_pair
    out = {}
    cases = []
    for k, (n, eps) in enumerate(((8, 1e-4), (16, 1e-5), (32, 1e-6), (48, 1e-6))):
        rng = np.random.Generator(np.random.Philox(3000 + k))
        a, u = make_instance(ref, rng, n)
        x = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
        kk = x - x.conj().T
        kk *= eps / np.linalg.norm(kk)
        poly = np.eye(n) + kk + kk @ kk / 2.0 + kk @ kk @ kk / 6.0
        qhat = matmul_hp(u, DDMatrix.from_lp(poly))
        pair, rep = refine_template(a, qhat, RefineConfig())
        v = verify_pair(a, pair)
        for name, mat in (("a", a), ("qhat", qhat), ("q", pair.q), ("t", pair.t)):
            for cell, arr in zip(("rh", "rl", "ih", "il"), mat.cells()):
                out["%s%s_%d" % (name, cell, k)] = np.ascontiguousarray(arr)
        cases.append(dict(k=k, n=n, eps=eps, iterations=rep.iterations, status=rep.status.value,
                          residual_history=[list(map(float, r)) for r in rep.residual_history],
                          hp_matmul_count=rep.hp_matmul_count, clipped_total=rep.clipped_total,
                          skip_fired=bool(rep.skip_fired), verify=list(map(float, v))))
    np.savez_compressed(os.path.join(HERE, "refine_dd_ref.npz"), **out)
    with open(os.path.join(HERE, "refine_dd_ref.json"), "w") as f:
        json.dump(dict(source="ddschur.refine.refine_template (refine.py:357-380), default RefineConfig",
                       cases=cases), f, indent=1)


def gen_configs(ref):
    """BASELINE configs the reference can run here:
    config 1 (n=256) through the reference as-is (dd hp, binary64 lp) with
    the FP64 stop rule re-expressed as tol_factor = 10 * 2^53 / n,
    max_iters = 10 (option 1); config 4 literal at n = 64 / 128 (dd mode,
    default stop) and its well-conditioned variant (strict part / sqrt(n))
    at n = 128."""
    from ddschur.refine import RefineConfig, refine_template
    from paper_2203_10879_b200 import inputs
    out = {}
    cases = []
    runs = []
    a1, q1 = inputs.config_inputs(1, 256)
    runs.append(("config1_n256", a1, q1, RefineConfig(tol_factor=10 * 2.0 ** 53 / 256, max_iters=10),
                 "option1: reference dd, tol_factor=10*2^53/n, max_iters=10"))
    for n, scale, tag in ((64, 1.0, "config4_n64"), (128, 1.0, "config4_n128"),
                          (128, None, "config4wc_n128")):
        s = 1.0 / np.sqrt(n) if scale is None else scale
        a = inputs.config4_matrix(n, 0, strict_scale=s)
        q = inputs.schur_vectors(a, np.complex128)
        runs.append((tag, a, q, RefineConfig(max_iters=10), "dd mode, default tol_factor=10, max_iters=10"))
    for tag, a, q, cfg, how in runs:
        t0 = time.time()
        try:
            pair, rep = refine_template(a, q, cfg)
            res = dict(iterations=rep.iterations, status=rep.status.value,
                       residual_history=[list(map(float, r)) for r in rep.residual_history],
                       hp_matmul_count=rep.hp_matmul_count, skip_fired=bool(rep.skip_fired),
                       detail=rep.detail)
        except Exception as exc:  # SeparationError etc. are results too
            res = dict(exception=type(exc).__name__, message=str(exc))
        res.update(tag=tag, n=int(a.shape[0]), how=how, seconds=time.time() - t0,
                   norm_a=float(np.linalg.norm(a)))
        out["qhat_" + tag] = q
        cases.append(res)
        print(tag, res.get("status"), res.get("iterations"), "%.1fs" % res["seconds"], flush=True)
    np.savez_compressed(os.path.join(HERE, "configs_ref.npz"), **out)
    with open(os.path.join(HERE, "configs_ref.json"), "w") as f:
        json.dump(dict(source="ddschur.refine.refine_template on BASELINE-config inputs", cases=cases), f,
                  indent=1)


def _digest(x):
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(x).tobytes()).hexdigest()[:16]


def _ref_case(tag, a, q, cfg, how, verify=False):
    from ddschur.refine import refine_template, verify_pair
    t0 = time.time()
    try:
        pair, rep = refine_template(a, q, cfg)
        res = dict(iterations=rep.iterations, status=rep.status.value,
                   residual_history=[list(map(float, r)) for r in rep.residual_history],
                   hp_matmul_count=rep.hp_matmul_count, skip_fired=bool(rep.skip_fired),
                   detail=rep.detail)
        if verify and rep.status.value == "Converged":
            res["verify"] = list(map(float, verify_pair(a, pair)))
    except Exception as exc:  # SeparationError etc. are results too
        res = dict(exception=type(exc).__name__, message=str(exc))
    res.update(tag=tag, n=int(a.shape[0]), how=how, seconds=time.time() - t0,
               norm_a=float(np.linalg.norm(a)), qhat_sha256_16=_digest(q))
    print(tag, res.get("status"), res.get("iterations"), "%.1fs" % res["seconds"], flush=True)
    return res


def gen_configs_full(ref):
    """BASELINE config 4 at its stated size n = 1024, in the reference's
    native dd mode (default tol_factor = 10, max_iters = 10): the literal
    matrix (the reference ends NonFinite) and the documented
    well-conditioned variant (strict part / sqrt(n)).  Q̂ = complex128 Schur
    vectors (zgees) — too large to commit (16 MiB), so the fixture records
    its digest and the tests rebuild it with the same LAPACK call."""
    from ddschur.refine import RefineConfig
    from paper_2203_10879_b200 import inputs
    cases = []
    for scale, tag in ((1.0, "config4_n1024"), (None, "config4wc_n1024")):
        n = 1024
        s = 1.0 / np.sqrt(n) if scale is None else scale
        a = inputs.config4_matrix(n, 0, strict_scale=s)
        q = inputs.schur_vectors(a, np.complex128)
        cases.append(_ref_case(tag, a, q, RefineConfig(max_iters=10), "dd mode, default tol_factor=10, "
                               "max_iters=10", verify=True))
    with open(os.path.join(HERE, "configs_full_ref.json"), "w") as f:
        json.dump(dict(source="ddschur.refine.refine_template (unmodified reference, dd mode) on BASELINE "
                              "config 4 at n=1024", cases=cases), f, indent=1)


def gen_config2(ref):
    """BASELINE config 2 (n = 2048 complex Gaussian, complex64-Schur start)
    through the unmodified reference (option 1: dd hp, binary64 lp) with the
    FP64 stop rule re-expressed as tol_factor = 10 * 2^53 / n, max_iters = 10.
    About 30 min on 8 cores; the result is the reference's own iteration
    count and status at the config's stated size."""
    from ddschur.refine import RefineConfig
    from paper_2203_10879_b200 import inputs
    a, q = inputs.config_inputs(2, 2048)
    n = 2048
    case = _ref_case("config2_n2048", a, q, RefineConfig(tol_factor=10 * 2.0 ** 53 / n, max_iters=10),
                     "option1: reference dd, tol_factor=10*2^53/n, max_iters=10")
    with open(os.path.join(HERE, "config2_ref.json"), "w") as f:
        json.dump(dict(source="ddschur.refine.refine_template (unmodified reference) on BASELINE config 2",
                       cases=[case]), f, indent=1)


def gen_ddops(ref):
    """DDMatrix arithmetic and the matrix-core helpers on seeded normalised
    dd inputs: a + b, a - b, a.scale(s), frobenius_norm(a) (hi, lo) and
    stril_extract(a) (ddmatrix.py:114-147, 190-251) — the pins of the
    bit-identical GPU versions (csrc/dd_ops.cu)."""
    from ddschur.ddmatrix import DDMatrix, frobenius_norm, stril_extract
    out = {}
    cases = []
    for k, (m, n) in enumerate(((5, 5), (37, 29), (64, 64), (61, 47))):
        rng = np.random.Generator(np.random.Philox(4000 + k))

        def dd():
            cells = []
            for _ in range(2):
                hi = rng.standard_normal((m, n)) * np.exp2(rng.integers(-30, 30, (m, n)))
                lo = hi * rng.standard_normal((m, n)) * 2.0 ** -60
                s_ = hi + lo
                cells += [s_, lo - (s_ - hi)]
            return DDMatrix(cells[0], cells[1], cells[2], cells[3])
        a, b = dd(), dd()
        s = float(rng.standard_normal() * 3.7)
        res = {"a": a, "b": b, "add": a + b, "sub": a - b, "scale": a.scale(s)}
        if m == n:
            e, t = stril_extract(a)
            res["stril_e"], res["stril_t"] = e, t
        for name, mat in res.items():
            for cell, arr in zip(("rh", "rl", "ih", "il"), mat.cells()):
                out["%s%s_%d" % (name, cell, k)] = np.ascontiguousarray(arr)
        nrm = frobenius_norm(a)
        cases.append(dict(k=k, m=m, n=n, s=s, norm_hi=float(nrm.hi), norm_lo=float(nrm.lo)))
    np.savez_compressed(os.path.join(HERE, "ddops_ref.npz"), **out)
    with open(os.path.join(HERE, "ddops_ref.json"), "w") as f:
        json.dump(dict(source="ddschur.ddmatrix DDMatrix +, -, scale, frobenius_norm, stril_extract", cases=cases),
                  f, indent=1)


def gen_symmetric(ref):
    """refine_symmetric (refine.py:409-438) in the reference's dd mode on
    seeded Hermitian matrices A = (X + X^H) / 2 (Philox), default config:
    status, iterations, history, hp count, detail, the refined T diagonal
    (dd) and verify_pair of the result; plus the NotSymmetric rejection."""
    from ddschur.refine import NotSymmetric, RefineConfig, refine_symmetric, verify_pair
    out = {}
    cases = []
    for k, n in enumerate((12, 24, 40)):
        rng = np.random.Generator(np.random.Philox(5000 + k))
        x = (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))) * np.sqrt(0.5)
        a = (x + x.conj().T) / 2.0
        pair, rep = refine_symmetric(a, RefineConfig(seed=k))
        v = verify_pair(a, pair)
        out["a_%d" % k] = a
        for cell, arr in zip(("rh", "rl", "ih", "il"), pair.t.cells()):
            out["t%s_%d" % (cell, k)] = np.ascontiguousarray(np.diag(arr))
        cases.append(dict(k=k, n=n, seed=k, iterations=rep.iterations, status=rep.status.value,
                          residual_history=[list(map(float, r)) for r in rep.residual_history],
                          hp_matmul_count=rep.hp_matmul_count, skip_fired=bool(rep.skip_fired),
                          detail=rep.detail, verify=list(map(float, v))))
    rng = np.random.Generator(np.random.Philox(5100))
    bad = rng.standard_normal((8, 8))
    try:
        refine_symmetric(bad)
        rejected = ""
    except NotSymmetric as exc:
        rejected = str(exc)
    out["a_nonsym"] = bad
    np.savez_compressed(os.path.join(HERE, "symmetric_ref.npz"), **out)
    with open(os.path.join(HERE, "symmetric_ref.json"), "w") as f:
        json.dump(dict(source="ddschur.refine.refine_symmetric (refine.py:409-438), RefineConfig(seed=k)",
                       cases=cases, nonsym_message=rejected), f, indent=1)


def gen_mixed(ref):
    """refine_mixed (refine.py:383-406) in the reference's dd mode on seeded
    complex Gaussian matrices (Philox), default config with seed k: status,
    iterations, history, hp count, the refined T diagonal (dd, in the
    random-line order) and verify_pair of the result."""
    from ddschur.refine import RefineConfig, refine_mixed, verify_pair
    out = {}
    cases = []
    for k, n in enumerate((12, 24, 40)):
        rng = np.random.Generator(np.random.Philox(6000 + k))
        a = (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))) * np.sqrt(0.5)
        pair, rep = refine_mixed(a, RefineConfig(seed=k))
        v = verify_pair(a, pair)
        out["a_%d" % k] = a
        for cell, arr in zip(("rh", "rl", "ih", "il"), pair.t.cells()):
            out["t%s_%d" % (cell, k)] = np.ascontiguousarray(np.diag(arr))
        cases.append(dict(k=k, n=n, seed=k, iterations=rep.iterations, status=rep.status.value,
                          residual_history=[list(map(float, r)) for r in rep.residual_history],
                          hp_matmul_count=rep.hp_matmul_count, skip_fired=bool(rep.skip_fired),
                          detail=rep.detail, verify=list(map(float, v))))
    np.savez_compressed(os.path.join(HERE, "mixed_ref.npz"), **out)
    with open(os.path.join(HERE, "mixed_ref.json"), "w") as f:
        json.dump(dict(source="ddschur.refine.refine_mixed (refine.py:383-406), RefineConfig(seed=k)",
                       cases=cases), f, indent=1)


def gen_io(ref):
    """Matrix Market files written by the reference (mmio.py:179-217) and the
    planes its reader returns (mmio.py:137-156), plus a coordinate symmetric
    file and a schema-v1 run record built by the reference (cli.py:83-103)."""
    from ddschur.ddmatrix import DDMatrix
    from ddschur.generators import MatrixKind, MatrixSpec
    from ddschur.mmio import read_matrix_market, write_matrix_market
    from ddschur.cli import build_run_record, validate_run_record
    from ddschur.refine import RefineConfig, refine_template, verify_pair
    rng = np.random.Generator(np.random.Philox(7000))
    out = {}
    n = 5
    hi = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    lo = (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))) * 1e-17
    dd = DDMatrix.from_lp(hi) + DDMatrix.from_lp(lo)
    write_matrix_market(os.path.join(HERE, "mm_dd_complex.mtx"), dd, comment="reference writer, dd")
    write_matrix_market(os.path.join(HERE, "mm_f64_real.mtx"), rng.standard_normal((3, 4)), comment="binary64")
    with open(os.path.join(HERE, "mm_coord_sym.mtx"), "w") as f:
        f.write("%%MatrixMarket matrix coordinate real symmetric\n% hand-written\n4 4 5\n"
                "1 1 2.5\n2 1 -1\n3 2 0.1\n4 4 1e-300\n4 3 3.14159265358979323846264338327950288\n")
    for tag in ("dd_complex", "f64_real", "coord_sym"):
        m = read_matrix_market(os.path.join(HERE, "mm_%s.mtx" % tag))
        for cell, arr in zip(("rh", "rl", "ih", "il"), m.cells()):
            out["%s_%s" % (tag, cell)] = np.ascontiguousarray(arr)
    for cell, arr in zip(("rh", "rl", "ih", "il"), dd.cells()):
        out["src_%s" % cell] = np.ascontiguousarray(arr)
    np.savez_compressed(os.path.join(HERE, "io_ref.npz"), **out)
    # a run record of a real refinement
    a = (rng.standard_normal((8, 8)) + 1j * rng.standard_normal((8, 8)))
    from ddschur.refine import refine_mixed
    pair, rep = refine_mixed(a, RefineConfig(seed=1))
    spec = MatrixSpec(kind=MatrixKind.RANDN_COMPLEX, n=8, seed=1)
    rec = validate_run_record(build_run_record(spec, RefineConfig(seed=1), rep, verify_pair(a, pair)))
    with open(os.path.join(HERE, "run_record_ref.json"), "w") as f:
        json.dump(rec, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    ref = import_reference()
    which = sys.argv[1:] or ["trisolve", "ddgemm", "refine_dd", "configs", "symmetric", "mixed", "io"]
    for w in which:
        t0 = time.time()
        globals()["gen_" + w](ref)
        print("generated", w, "%.1fs" % (time.time() - t0), flush=True)
