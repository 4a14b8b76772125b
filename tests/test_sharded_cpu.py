"""Multi-process host logic of the sharded driver on CPU (gloo, world_size 2):
partitions are disjoint and complete, and the gathered output equals the
single-process oracle result.  The compute step is the oracle's exact GEMM
(the GPU kernels are covered by the -m gpu tests)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2210_16691_b200.sharded import all_shards, shard_range


@pytest.mark.parametrize("total,world,granule", [(4096, 2, 128), (4096, 8, 128), (300, 3, 128), (192, 8, 1),
                                                 (5, 8, 1), (0, 2, 1), (1000, 7, 128)])
def test_partition_disjoint_and_complete(total, world, granule):
    shards = all_shards(total, world, granule)
    covered = []
    for s in shards:
        assert s.start <= s.stop
        if s.size and s.stop < total:
            assert s.size % granule == 0
        covered.extend(range(s.start, s.stop))
    assert covered == list(range(total))
    granules = [-(-s.size // granule) for s in shards]
    assert max(granules) - min(granules) <= 1


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import coracle
        from oracle.splitmix import gemm_inputs
        from paper_2210_16691_b200.sharded import batch_sharded, m_sharded_matmul

        a, b = gemm_inputs(300, 64, 96, seed=5)
        A, B = torch.from_numpy(a), torch.from_numpy(b)
        full, sh = m_sharded_matmul(A, B, rank, world, compute=lambda x, y: torch.from_numpy(
            coracle.gemm_i64(x.numpy(), y.numpy())), gather=True)
        ref = torch.from_numpy(coracle.gemm_i64(a, b))
        ok_m = bool(torch.equal(full, ref))
        # batch sharding (BMM / conv images)
        xa, xb = gemm_inputs(32, 16, 24, batch=5, seed=9)
        X = torch.from_numpy(xa)
        Y = torch.from_numpy(xb)
        gathered, _ = batch_sharded(lambda xs: torch.from_numpy(
            coracle.gemm_i64(xs.numpy(), Y[:xs.shape[0]].numpy() * 0 + Y[0].numpy())), X, rank, world, gather=True)
        ref_b = torch.from_numpy(coracle.gemm_i64(xa, np.broadcast_to(xb[0], xb.shape).copy()))
        ok_b = bool(torch.equal(gathered, ref_b))
        # 256-row granules (the bench's square GEMM shards), uneven: 700 rows over 2 ranks
        from paper_2210_16691_b200.sharded import gather_rows, shard_range
        rows = torch.arange(700 * 3, dtype=torch.float32).view(700, 3)
        s256 = shard_range(700, rank, world, granule=256)
        g256 = gather_rows(rows[s256.start:s256.stop].clone(), 700, rank, world, granule=256)
        ok_b = ok_b and bool(torch.equal(g256, rows))
        # max-over-ranks timing reduction
        t = torch.tensor([float(rank + 1)])
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        out[rank] = (ok_m, ok_b, float(t.item()), sh.start, sh.stop)
    finally:
        dist.destroy_process_group()


def test_gloo_two_ranks_gather_equals_oracle():
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    assert len(out) == world
    for r in range(world):
        ok_m, ok_b, tmax, start, stop = out[r]
        assert ok_m and ok_b
        assert tmax == float(world)
    assert out[0][3] == 0 and out[0][4] == out[1][3] and out[1][4] == 300


@pytest.mark.parametrize("total,world,granule", [(16384, 8, 256), (4096, 3, 256), (1000, 4, 128), (192, 8, 1),
                                                 (256, 5, 1), (7, 8, 1), (0, 2, 1), (300, 2, 256)])
def test_abi_shard_range_matches_python(total, world, granule):
    """alcop_shard_range (the C ABI multi-GPU driver's split) == sharded.shard_range (bench / gloo tests)."""
    import paper_2210_16691_b200 as alcop
    from paper_2210_16691_b200.sharded import shard_range
    for r in range(world):
        sh = shard_range(total, r, world, granule)
        assert alcop.shard_range(total, r, world, granule) == (sh.start, sh.size)


def test_abi_sharded_rejects_bad_shards():
    import ctypes
    import paper_2210_16691_b200 as alcop
    lib = alcop.load_library()
    d = alcop.gemm_desc(1024, 1024, 1024)
    assert lib.alcop_gemm_sharded(ctypes.byref(d), None, 0, None, 256) == alcop.ALCOP_ERR_CONFIG
    assert lib.alcop_last_error().decode().startswith("BadShards")
    arr = (alcop.Shard * 1)(alcop.Shard(99, None, 16, 16, 16))
    assert lib.alcop_gemm_sharded(ctypes.byref(d), None, 1, arr, 256) == alcop.ALCOP_ERR_CUDA
    d.ldc = 2048
    assert lib.alcop_gemm_sharded(ctypes.byref(d), None, 1, arr, 256) == alcop.ALCOP_ERR_CONFIG
