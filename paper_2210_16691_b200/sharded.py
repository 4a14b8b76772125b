"""Batch / M-sharded multi-GPU driver.

One process per GPU (torchrun), ``torch.distributed`` for the plumbing.  The
pipelined GEMM path partitions cleanly: independent batches (BMM, conv
images) or disjoint row blocks of C (large square GEMMs, B replicated), so
the compute path has no collective.  NCCL appears only in the optional
all-gather of the output shards (over NVLink/NVSwitch), timed separately, and
in the max-over-ranks timing.

The compute callable is injected (default: the sm_100a kernels through the C
ABI) so the partition/gather logic is testable with gloo on CPU.
"""
from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class Shard:
    rank: int
    world: int
    start: int  # first unit (row / batch index) owned by this rank
    stop: int   # one past the last

    @property
    def size(self) -> int:
        return self.stop - self.start


def shard_range(total: int, rank: int, world: int, granule: int = 1) -> Shard:
    """Contiguous split of `total` units over `world` ranks in multiples of
    `granule` (128 rows = one output tile row for M-sharding, 1 for batch).
    Earlier ranks take the remainder granules; every unit has one owner."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    g = -(-total // granule)  # granules
    base, extra = divmod(g, world)
    first = rank * base + min(rank, extra)
    count = base + (1 if rank < extra else 0)
    start = min(total, first * granule)
    stop = min(total, (first + count) * granule)
    return Shard(rank, world, start, stop)


def all_shards(total: int, world: int, granule: int = 1):
    return [shard_range(total, r, world, granule) for r in range(world)]


def m_sharded_matmul(A, B, rank, world, compute=None, sched=None, gather=False, group=None):
    """C = A @ B with the rows of A/C split over ranks (B replicated).
    Returns (C_local, shard) or the gathered C if gather=True."""
    import torch
    M = A.shape[-2]
    sh = shard_range(M, rank, world, granule=128)
    if compute is None:
        import paper_2210_16691_b200 as alcop

        def compute(a, b):
            return alcop.matmul(a, b, sched)
    local = compute(A[..., sh.start:sh.stop, :], B) if sh.size else A.new_empty((0, B.shape[-1]))
    if not gather:
        return local, sh
    return gather_rows(local, M, rank, world, group=group), sh


def batch_sharded(fn, X, rank, world, gather=False, group=None):
    """Applies fn to this rank's slice of the leading (batch) dimension."""
    sh = shard_range(X.shape[0], rank, world, granule=1)
    local = fn(X[sh.start:sh.stop])
    if not gather:
        return local, sh
    return gather_rows(local, X.shape[0], rank, world, group=group, dim0=True), sh


def gather_rows(local, total, rank, world, group=None, dim0=False, granule=None):
    """All-gathers uneven row shards (NCCL on GPU, gloo on CPU): pads every
    shard to the largest, gathers, then trims and concatenates in rank order.
    `granule` must be the one the rows were sharded with (default 1 for
    dim0 / batch, 128 for M rows)."""
    import torch
    import torch.distributed as dist
    shards = all_shards(total, world, granule or (1 if dim0 else 128))
    axis = 0 if dim0 else local.dim() - 2
    maxn = max(s.size for s in shards)
    pad_shape = list(local.shape)
    pad_shape[axis] = maxn
    buf = local.new_zeros(pad_shape)
    buf.narrow(axis, 0, local.shape[axis]).copy_(local)
    outs = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(outs, buf, group=group)
    return torch.cat([o.narrow(axis, 0, s.size) for o, s in zip(outs, shards)], dim=axis)
