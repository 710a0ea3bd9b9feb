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
    """Same protocol as sharded.OzakiShardBackend; complex128 products on the
    CPU (lp products in complex64), column blocks, partial norms all-reduced."""

    def __init__(self, a, qhat):
        self.a = torch.from_numpy(np.asarray(a, dtype=np.complex128))
        self.qhat = torch.from_numpy(np.asarray(qhat, dtype=np.complex128))
        self.n = self.a.shape[0]
        n = self.n
        self.q = torch.zeros((n, n), dtype=torch.complex128)
        self.t_full = torch.zeros((n, n), dtype=torch.complex128)
        self.x = torch.zeros((n, n), dtype=torch.complex64)

    def set_columns(self, j0, j1, ranges, group):
        self.j0, self.j1, self.ranges, self.group = j0, j1, ranges, group
        self.gather = parallel.ColGatherer(ranges, group)
        self.eye_j = torch.eye(self.n, dtype=torch.complex128)[:, j0:j1]

    def _gather(self, local, full):
        if full.is_complex():
            self.gather(torch.view_as_real(local.contiguous()), torch.view_as_real(full))
        else:
            self.gather(local.contiguous(), full)

    def _sum(self, values):
        return parallel.all_reduce_sum(values, torch.device("cpu"), self.group)

    def norm_guard(self):
        pass

    def entry_cols(self):
        j0, j1 = self.j0, self.j1
        yj = self.qhat.conj().T @ self.qhat[:, j0:j1] - self.eye_j
        self._sum([float(torch.linalg.matrix_norm(yj)) ** 2])  # the correction-plan bound (a collective)
        self.qj = self.qhat[:, j0:j1] - 0.5 * (self.qhat @ yj)

    def gather_q(self):
        self._gather(self.qj, self.q)

    def norm_a(self):
        return float(torch.linalg.matrix_norm(self.a))

    def measure_cols(self):
        j0, j1 = self.j0, self.j1
        qj = self.q[:, j0:j1]
        self.tj = self.q.conj().T @ (self.a @ qj)
        self.yj = self.q.conj().T @ qj - self.eye_j
        rows = torch.arange(self.n)[:, None]
        cols = torch.arange(j0, j1)[None, :]
        self.ej = torch.where(rows > cols, self.tj, torch.zeros_like(self.tj))

    def norms(self):
        se, sy = self._sum([float(torch.linalg.matrix_norm(self.ej)) ** 2,
                            float(torch.linalg.matrix_norm(self.yj)) ** 2])
        return float(np.sqrt(se)), float(np.sqrt(sy))

    def gather_lp(self):
        self._gather(self.tj, self.t_full)

    def solve(self, clip):
        t = torch.triu(self.t_full).numpy().astype(np.complex64)
        e = torch.tril(self.t_full, -1).numpy().astype(np.complex64)
        l, nclip = clib.solve_block(t, e, clip_threshold=clip, dtype=np.complex64)
        self.w = torch.from_numpy(l - l.conj().T)
        return float(np.linalg.norm(self.w.numpy().astype(np.complex128))), 0, nclip

    def update_cols(self, norm_y, norm_w):
        j0, j1 = self.j0, self.j1
        c = torch.complex128
        wj = self.w[:, j0:j1]
        w2j = self.w @ wj
        xj = (self.yj - wj.to(c) - w2j.to(c)).to(torch.complex64)  # X = Y - W - W^2
        self._gather(xj, self.x)
        xwj = self.x @ wj                                             # (X W)_J = (YW - W^2 - W^3)_J
        s = (2.0 * wj.to(c) - self.yj) - xwj.to(c)                    # S'_J
        self.qj = self.q[:, j0:j1] + 0.5 * (self.q @ s)

    def result(self):
        return self.q.clone(), torch.triu(self.t_full)


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


def test_column_ranges_never_empty():
    """n = 512 on 8 ranks at align 128 (config 5's size) must not
    leave a rank without columns (it would encode nothing while the others
    wait in a collective)."""
    for n in list(range(8, 600)) + [512, 1000, 2048, 8192]:
        for world in (2, 3, 4, 8):
            r = parallel.column_ranges(n, world, 128)
            assert len(r) == world and r[0][0] == 0 and r[-1][1] == n
            assert all(j1 > j0 for j0, j1 in r), (n, world, r)
            assert all(r[k][1] == r[k + 1][0] for k in range(world - 1))
    assert parallel.column_ranges(512, 8, 128) == [(64 * k, 64 * (k + 1)) for k in range(8)]
    with pytest.raises(ValueError):
        parallel.column_ranges(3, 8)


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
