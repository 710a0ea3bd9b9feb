"""World-size-2 gloo tests (CPU) of the multi-GPU path's host logic:
column sharding, all-gathers, norm reductions and the sharded refinement
driver (paper_2203_10879_b200/sharded.py), run with a reference-arithmetic
backend (numpy-equivalent complex128 products on torch CPU tensors + the C
oracle solver) so the whole distributed control flow is exercised without a
GPU.  The result must equal the single-process oracle run on the same input."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import clib
from oracle.refine_fp64 import refine_template_fp64
from paper_2203_10879_b200 import parallel
from paper_2203_10879_b200.refine import RefineConfig

U = 2.0 ** -53


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class CpuShardBackend:
    """Same protocol as sharded.OzakiShardBackend; complex128 products on the CPU."""

    def __init__(self, a, qhat):
        self.a = torch.from_numpy(np.asarray(a, dtype=np.complex128))
        self.qhat = torch.from_numpy(np.asarray(qhat, dtype=np.complex128))
        self.n = self.a.shape[0]
        n = self.n
        self.q = torch.zeros((n, n), dtype=torch.complex128)
        self.that = torch.zeros_like(self.q)
        self.y = torch.zeros_like(self.q)
        self.w2 = torch.zeros((n, n), dtype=torch.complex64)

    def set_columns(self, j0, j1, ranges, group):
        self.j0, self.j1, self.ranges, self.group = j0, j1, ranges, group

    def _gather(self, local, full):
        if full.is_complex():
            parallel.all_gather_cols(torch.view_as_real(local), torch.view_as_real(full), self.ranges, self.group)
        else:
            parallel.all_gather_cols(local, full, self.ranges, self.group)

    def norm_guard(self):
        pass

    def entry_cols(self):
        j0, j1 = self.j0, self.j1
        eye = torch.eye(self.n, dtype=torch.complex128)[:, j0:j1]
        yj = self.qhat.conj().T @ self.qhat[:, j0:j1] - eye
        self.qj = self.qhat[:, j0:j1] - 0.5 * (self.qhat @ yj)

    def gather_q(self):
        self._gather(self.qj.contiguous(), self.q)

    def norm_a(self):
        return float(torch.linalg.matrix_norm(self.a))

    def measure_cols(self):
        j0, j1 = self.j0, self.j1
        qj = self.q[:, j0:j1]
        self.tj = self.q.conj().T @ (self.a @ qj)
        self.yj = self.q.conj().T @ qj - torch.eye(self.n, dtype=torch.complex128)[:, j0:j1]

    def gather_that_y(self):
        self._gather(self.tj.contiguous(), self.that)
        self._gather(self.yj.contiguous(), self.y)

    def norms(self):
        e = torch.tril(self.that, -1)
        return float(torch.linalg.matrix_norm(e)), float(torch.linalg.matrix_norm(self.y))

    def solve(self, clip):
        t = torch.triu(self.that).numpy().astype(np.complex64)
        e = torch.tril(self.that, -1).numpy().astype(np.complex64)
        l, nclip = clib.solve_block(t, e, clip_threshold=clip, dtype=np.complex64)
        self.w = torch.from_numpy(l - l.conj().T)
        return float(np.linalg.norm(self.w.numpy().astype(np.complex128))), 0, nclip

    def update_stage1_cols(self):
        j0, j1 = self.j0, self.j1
        y_lp = self.y.to(torch.complex64)
        wj = self.w[:, j0:j1]
        self.ywj = y_lp @ wj
        self.w2j = self.w @ wj

    def gather_w2(self):
        self._gather(self.w2j.contiguous(), self.w2)

    def update_stage2_cols(self):
        j0, j1 = self.j0, self.j1
        wj = self.w[:, j0:j1]
        w3j = self.w2 @ wj
        c = torch.complex128
        s = ((2.0 * wj.to(c) - self.y[:, j0:j1]) - self.ywj.to(c)) + self.w2j.to(c)
        s = s + w3j.to(c)
        self.qj = self.q[:, j0:j1] + 0.5 * (self.q @ s)

    def result(self):
        return self.q.clone(), torch.triu(self.that)


def _worker(rank, world, port, n, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2203_10879_b200 import inputs, sharded
        a = inputs.gaussian_complex(n, 3)
        q = inputs.schur_vectors(a).astype(np.complex128)
        be = CpuShardBackend(a, q)
        cfg = RefineConfig(precision="fp64", tol_factor=10.0 / n, max_iters=10)
        qf, tf, rep = sharded.refine_sharded(be, cfg, align=8)
        out[rank] = (qf.numpy(), rep["iterations"], rep["status"].value,
                     [tuple(h) for h in rep["residual_history"]], be.j0, be.j1)
    finally:
        dist.destroy_process_group()


def test_column_ranges():
    assert parallel.column_ranges(8192, 1) == [(0, 8192)]
    r = parallel.column_ranges(8192, 8)
    assert r[0] == (0, 1024) and r[-1] == (7168, 8192)
    r = parallel.column_ranges(1000, 3, align=128)
    assert r == [(0, 384), (384, 768), (768, 1000)]
    assert all(j0 % 128 == 0 for j0, _ in r)


def test_sharded_refinement_gloo_world2_matches_single_process():
    n, world = 48, 2
    mgr = mp.Manager()
    out = mgr.dict()
    port = free_port()
    mp.spawn(_worker, args=(world, port, n, out), nprocs=world, join=True)
    from paper_2203_10879_b200 import inputs
    a = inputs.gaussian_complex(n, 3)
    q = inputs.schur_vectors(a).astype(np.complex128)
    ref = refine_template_fp64(a, q, tol_factor=10.0 / n, max_iters=10)
    q0, it0, st0, h0, a0, b0 = out[0]
    q1, it1, st1, h1, a1, b1 = out[1]
    assert (a0, b0, a1, b1) == (0, 24, 24, 48)           # both ranks own half the columns
    assert np.array_equal(q0, q1) and h0 == h1            # replicated state is identical
    assert it0 == ref["iterations"] and st0 == ref["status"] == "Converged"
    assert np.abs(q0 - ref["q"]).max() <= 1e-13
    # the sharded products associate as Q^H (A Q) instead of (Q^H A) Q: the
    # histories agree to the lp (complex64) level of the correction
    for (e, y), (er, yr) in zip(h0, ref["residual_history"]):
        assert abs(e - er) <= 1e-2 * er + 100 * U * n
    assert h0[-1][0] <= 10 * U * np.linalg.norm(a)
