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
