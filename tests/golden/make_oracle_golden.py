"""Golden runs of the CPU restatement (oracle/refine_fp64.py) at the BASELINE
configs' stated sizes, for the FP64 mode the reference does not have
("parity unpinned by reference tests — pin it with golden
runs from both oracles on the §8d inputs, stored as JSON").

    python tests/golden/make_oracle_golden.py [config2] [config3] [config5]

config2: n = 2048 complex Gaussian, complex64-Schur start (C solver).
config3: n = 8192 real Gaussian, complex64-Schur start — the bench
         workload; the BLAS-backed solver port (oracle/trisolve_blas.py,
         pinned to the C restatement in tests/test_oracle.py), ~10 min here.
config5: the 64-step n = 512 continuation chain A(t_j) = A0 + t_j A1,
         t_j = 0.01 j / 64, each step started from the previous refined Q
         (C solver).

Q̂ is LAPACK cgees output, rebuilt by the tests with the same call
(paper_2203_10879_b200.inputs); each case records its digest.
"""
import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)

from oracle.refine_fp64 import refine_template_fp64, residuals_fp64  # noqa: E402
from paper_2203_10879_b200 import inputs  # noqa: E402


def digest(x):
    return hashlib.sha256(np.ascontiguousarray(x).tobytes()).hexdigest()[:16]


def summary(out, a, q0, tag, seconds, solver, evaluate=True):
    res = dict(tag=tag, n=int(a.shape[0]), status=out["status"], iterations=out["iterations"],
               residual_history=[list(map(float, r)) for r in out["residual_history"]],
               hp_matmul_count=out["hp_matmul_count"], skip_fired=bool(out["skip_fired"]),
               norm_a=out["norm_a"], seconds=seconds, solver=solver, qhat_sha256_16=digest(q0))
    if evaluate:
        rel_e, ortho = residuals_fp64(a, out["q"])
        res.update(final_rel_e=rel_e, final_ortho=ortho)
    print(tag, res["status"], res["iterations"], "%.1fs" % seconds, flush=True)
    return res


def gen_config2():
    a, q = inputs.config_inputs(2)
    n = a.shape[0]
    t0 = time.time()
    out = refine_template_fp64(a, q, tol_factor=10.0 / n, max_iters=10)
    return [summary(out, a, q, "config2_n2048", time.time() - t0, "c")]


def gen_config3():
    a, q = inputs.config_inputs(3)
    n = a.shape[0]
    t0 = time.time()
    out = refine_template_fp64(a, q, tol_factor=10.0 / n, max_iters=10, solver="blas")
    return [summary(out, a, q, "config3_n8192", time.time() - t0, "blas")]


def gen_config5(n=512, steps=64):
    a0, a1 = inputs.config5_pair(n, 0)
    q0 = inputs.schur_vectors(a0).astype(np.complex128)
    q = q0
    chain = []
    t0 = time.time()
    for j in range(steps):
        tj = 0.01 * j / 64
        a = a0 + tj * a1
        ts = time.time()
        out = refine_template_fp64(a, q, tol_factor=10.0 / n, max_iters=10)
        s = summary(out, a, q, "config5_step%02d" % j, time.time() - ts, "c")
        s["t"] = tj
        chain.append(s)
        q = out["q"]
    print("config5 chain %.1fs" % (time.time() - t0), flush=True)
    return [dict(tag="config5_chain_n512", n=n, steps=steps, qhat0_sha256_16=digest(q0), chain=chain)]


if __name__ == "__main__":
    which = sys.argv[1:] or ["config2", "config5", "config3"]
    for w in which:
        cases = globals()["gen_" + w]()
        with open(os.path.join(HERE, "oracle_%s.json" % w), "w") as f:
            json.dump(dict(source="oracle/refine_fp64.py (CPU restatement of refine.py:223-329 in FP64 mode) on "
                                  "BASELINE %s inputs, tol_factor=10/n, max_iters=10" % w, cases=cases), f, indent=1)
