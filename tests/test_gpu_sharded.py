"""The sharded (multi-GPU) driver on the GPU with a world of one rank: the
same column-sharded code path (sharded.OzakiShardBackend, NCCL collectives on
a size-1 group) must reproduce the single-GPU refinement.  Multi-rank runs
are covered on the CPU by tests/test_parallel.py (gloo); this run has one
GPU, and ranks that wait on each other must not share a GPU."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist

from oracle.refine_fp64 import refine_template_fp64, residuals_fp64
from paper_2203_10879_b200 import RefineConfig, inputs, refine_template
from paper_2203_10879_b200.sharded import refine_template_distributed

pytestmark = pytest.mark.gpu
U = 2.0 ** -53


def test_sharded_driver_world1_matches_single_gpu():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        n = 256
        a = inputs.gaussian_real(n, 2)
        q = inputs.schur_vectors(a).astype(np.complex128)
        cfg = RefineConfig(precision="fp64", tol_factor=10.0 / n, max_iters=10)
        pair, rep = refine_template_distributed(a, q, cfg)
        pair1, rep1 = refine_template(a, q, cfg)
        ref = refine_template_fp64(a, q, tol_factor=10.0 / n, max_iters=10)
        assert rep.status.value == rep1.status.value == ref["status"] == "Converged"
        assert abs(rep.iterations - ref["iterations"]) <= 1 and rep.iterations == rep1.iterations
        assert rep.hp_matmul_count == rep1.hp_matmul_count
        rel_e, ortho = residuals_fp64(a, pair.q.cpu().numpy())
        assert rel_e <= 15 * U and ortho <= 2 * max(residuals_fp64(a, ref["q"])[1], 10 * np.sqrt(n) * U)
    finally:
        dist.destroy_process_group()


def _nccl_worker(rank, world, port, n, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world)
    try:
        a = inputs.gaussian_real(n, 2)
        q = inputs.schur_vectors(a).astype(np.complex128)
        cfg = RefineConfig(precision="fp64", tol_factor=10.0 / n, max_iters=10)
        pair, rep = refine_template_distributed(a, q, cfg)
        out[rank] = (pair.q.cpu().numpy(), rep.iterations, rep.status.value, rep.residual_history,
                     rep.hp_matmul_count)
    finally:
        dist.destroy_process_group()


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs two GPUs (one process per GPU)")
def test_sharded_driver_world2_nccl_matches_single_gpu():
    """Two ranks on two GPUs over NCCL: identical replicated state on both
    ranks and the single-GPU result (skipped on a one-GPU box: ranks that
    wait on each other must not share a GPU)."""
    import torch.multiprocessing as mp
    n, world = 512, 2
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    out = mp.Manager().dict()
    mp.spawn(_nccl_worker, args=(world, port, n, out), nprocs=world, join=True)
    a = inputs.gaussian_real(n, 2)
    q = inputs.schur_vectors(a).astype(np.complex128)
    cfg = RefineConfig(precision="fp64", tol_factor=10.0 / n, max_iters=10)
    pair1, rep1 = refine_template(a, q, cfg)
    q0, it0, st0, h0, hp0 = out[0]
    q1, it1, st1, h1, hp1 = out[1]
    assert np.array_equal(q0, q1) and h0 == h1
    assert st0 == rep1.status.value == "Converged" and it0 == rep1.iterations and hp0 == rep1.hp_matmul_count
    rel_e, ortho = residuals_fp64(a, q0)
    assert rel_e <= 15 * U
