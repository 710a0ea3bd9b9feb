"""Collectives and sharding for the multi-GPU refinement (one process per GPU).

The sharded driver (sharded.py) splits every product by output COLUMNS:
rank r owns columns J_r of T^, Y, Sigma' and Q_new, while A, Q and the lp
matrices the solver needs are replicated.  With A and Q resident on every
rank, T^[:, J] = Q^H (A Q[:, J]) and Y[:, J] = Q^H Q[:, J] - I need no
exchange; the exchanges per iteration are all-gathers of
column blocks (lp T^ for the solver, lp Y and W^2 for the merged update,
Q_new in hp) and one all-reduce of the partial norms.  Everything here runs
on torch tensors through torch.distributed, so the same code drives NCCL on
the GPUs and gloo in the CPU tests.
"""
import torch
import torch.distributed as dist


def column_ranges(n, world, align=128):
    """[(j0, j1)] per rank: contiguous column blocks, widths multiples of
    `align` (the Ozaki GEMM's tile) except possibly the last one.  Every rank
    gets at least one column: when world * align would leave ranks empty
    (n = 512 on 8 ranks at align 128) the alignment is halved until none is
    (an empty rank would encode nothing while the others wait in a
    collective)."""
    if world <= 1:
        return [(0, n)]
    if n < world:
        raise ValueError("cannot shard %d columns over %d ranks" % (n, world))
    while True:
        per = -(-n // world)
        per = -(-per // align) * align
        if (world - 1) * per < n:
            break
        if align == 1:  # balanced widths n // world (+1 for the first n % world ranks)
            base, extra = divmod(n, world)
            bounds = [r * base + min(r, extra) for r in range(world + 1)]
            return [(bounds[r], bounds[r + 1]) for r in range(world)]
        align //= 2
    out = []
    for r in range(world):
        j0 = min(n, r * per)
        j1 = min(n, j0 + per)
        out.append((j0, j1))
    return out


def world_info(group=None):
    if not dist.is_available() or not dist.is_initialized():
        return 0, 1
    return dist.get_rank(group), dist.get_world_size(group)


def all_gather_cols(local, full, ranges, group=None):
    """Gather column blocks into `full` on every rank.

    local: (rows, w_r, *extra) tensor of this rank's block (any strides);
    full:  (rows, >= n, *extra) destination (columns j0..j1 of rank r <- its block).
    Blocks are padded to the widest so one all_gather_into_tensor moves them."""
    rank, world = world_info(group)
    if world == 1:
        j0, j1 = ranges[0]
        if full[:, j0:j1].data_ptr() != local.data_ptr():
            full[:, j0:j1].copy_(local)
        return full
    wmax = max(j1 - j0 for j0, j1 in ranges)
    rows = local.shape[0]
    extra = tuple(local.shape[2:])
    send = torch.zeros((rows, wmax) + extra, dtype=local.dtype, device=local.device)
    send[:, : local.shape[1]].copy_(local)
    recv_flat = torch.empty((world * rows, wmax) + extra, dtype=local.dtype, device=local.device)
    dist.all_gather_into_tensor(recv_flat, send, group=group)  # rank-major concatenation
    recv = recv_flat.view((world, rows, wmax) + extra)
    for r, (j0, j1) in enumerate(ranges):
        if j1 > j0:
            full[:, j0:j1].copy_(recv[r, :, : j1 - j0])
    return full


class ColGatherer:
    """all_gather_cols with persistent buffers: one (rows, wmax, *extra)
    send buffer and one (world * rows, wmax, *extra) receive buffer, allocated
    once per shape (the driver gathers the same block shapes every
    iteration), so a gather allocates and zero-fills nothing."""

    def __init__(self, ranges, group=None):
        self.ranges, self.group = ranges, group
        self.rank, self.world = world_info(group)
        self.wmax = max(j1 - j0 for j0, j1 in ranges)
        self.bufs = {}

    def __call__(self, local, full):
        if self.world == 1:
            j0, j1 = self.ranges[0]
            if full[:, j0:j1].data_ptr() != local.data_ptr():
                full[:, j0:j1].copy_(local)
            return full
        rows = local.shape[0]
        extra = tuple(local.shape[2:])
        key = (rows, extra, local.dtype, local.device)
        if key not in self.bufs:
            self.bufs[key] = (torch.zeros((rows, self.wmax) + extra, dtype=local.dtype, device=local.device),
                              torch.empty((self.world * rows, self.wmax) + extra, dtype=local.dtype,
                                          device=local.device))
        send, recv_flat = self.bufs[key]
        send[:, : local.shape[1]].copy_(local)
        dist.all_gather_into_tensor(recv_flat, send, group=self.group)
        recv = recv_flat.view((self.world, rows, self.wmax) + extra)
        for r, (j0, j1) in enumerate(self.ranges):
            if j1 > j0:
                full[:, j0:j1].copy_(recv[r, :, : j1 - j0])
        return full


def all_reduce_sum(values, device, group=None):
    """Sum a short list of floats over the ranks (partial squared norms)."""
    _, world = world_info(group)
    t = torch.tensor(values, dtype=torch.float64, device=device)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return [float(v) for v in t.cpu()]


def all_reduce_max(values, device, group=None):
    _, world = world_info(group)
    t = torch.tensor(values, dtype=torch.float64, device=device)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return [float(v) for v in t.cpu()]
