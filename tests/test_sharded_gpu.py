"""The C-ABI multi-GPU driver (alcop_gemm_sharded / alcop_conv2d_sharded,
SURVEY §8e): one host thread per shard, each enqueueing its shard's launch on
its own device and stream.  This box has one GPU, so the shards name device 0
with distinct streams (the shard arithmetic, the per-thread launch and the
error plumbing are the same code as on N devices); results must equal the
exact product / direct conv bit for bit, empty shards included."""
import numpy as np
import pytest

from oracle import coracle

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _bf16(a):
    return torch.from_numpy(a).cuda().to(torch.bfloat16)


def _exact_rows(a, b):
    return coracle.gemm_rows_i8(a, b, np.arange(a.shape[0] if a.ndim == 2 else a.shape[0] * a.shape[1]))


@pytest.mark.parametrize("M,N,K,nshards,granule,sched", [
    (4096, 2048, 1024, 4, 256, None), (4096, 2048, 1024, 3, 256, "pair"), (1000, 768, 512, 4, 128, "single"),
    (256, 512, 256, 4, 256, None), (16384, 1024, 512, 8, 256, None)])
def test_gemm_m_sharded_exact(alcop, M, N, K, nshards, granule, sched):
    a = coracle.random_i8(M * K, 0).reshape(M, K)
    b = coracle.random_i8(K * N, 1).reshape(K, N)
    s = {None: None, "pair": alcop.make_schedule(tileN=256, tileK=64, n_stage=4, cta_group=2),
         "single": alcop.make_schedule(tileN=128, tileK=64, n_stage=4)}[sched]
    A, B = _bf16(a), _bf16(b)
    C = torch.full((M, N), float("nan"), device="cuda", dtype=torch.float32)
    streams = [torch.cuda.Stream() for _ in range(nshards)]
    shards = []
    for r in range(nshards):
        start, count = alcop.shard_range(M, r, nshards, granule)
        shards.append((0, streams[r], A[start:start + count] if count else None, B,
                       C[start:start + count] if count else None))
    d = alcop.gemm_desc(M, N, K, 1, alcop.BF16, alcop.F32, alcop.B_KN)
    alcop.gemm_sharded(d, shards, s, granule)
    torch.cuda.synchronize()
    assert np.array_equal(C.cpu().numpy().astype(np.int64), _exact_rows(a, b))


def test_bmm_batch_sharded_exact(alcop):
    bt, M, N, K = 192, 512, 512, 64
    a = coracle.random_i8(bt * M * K, 0).reshape(bt, M, K)
    b = coracle.random_i8(bt * K * N, 1).reshape(bt, K, N)
    A, B = _bf16(a), _bf16(b)
    C = torch.zeros((bt, M, N), device="cuda", dtype=torch.bfloat16)
    shards = []
    for r in range(5):
        start, count = alcop.shard_range(bt, r, 5, 1)
        shards.append((0, torch.cuda.Stream(), A[start:start + count], B[start:start + count],
                       C[start:start + count]))
    alcop.gemm_sharded(alcop.gemm_desc(M, N, K, bt, alcop.BF16, alcop.BF16, alcop.B_KN), shards, None, 1)
    torch.cuda.synchronize()
    want = coracle.to_f32(coracle.to_dtype(_exact_rows(a, b).reshape(bt, M, N).astype(np.float32), "bf16"), "bf16")
    assert np.array_equal(C.float().cpu().numpy(), want)


def test_conv_batch_sharded_exact(alcop):
    N, H, W, C, K, R = 7, 28, 28, 64, 128, 3
    x = coracle.random_i8(N * H * W * C, 21).reshape(N, H, W, C)
    w = coracle.random_i8(K * R * R * C, 22).reshape(K, R, R, C)
    X, Wt = _bf16(x), _bf16(w)
    Y = torch.full((N, H, W, K), float("nan"), device="cuda", dtype=torch.float32)
    s = alcop.make_schedule(tileN=128, tileK=64, n_stage=4)
    shards = []
    for r in range(4):
        start, count = alcop.shard_range(N, r, 4, 1)
        shards.append((0, torch.cuda.Stream(), X[start:start + count], Wt, Y[start:start + count]))
    d = alcop.conv_desc(N, H, W, C, K, R, R, (1, 1), (1, 1), alcop.BF16, alcop.F32)
    alcop.conv2d_sharded(d, s, shards)
    torch.cuda.synchronize()
    pts = np.array([(n, p, q) for n in range(N) for p in range(H) for q in range(W)], dtype=np.int64)
    want = coracle.conv2d_points_i8(x, w, (1, 1), (1, 1), pts).reshape(N, H, W, K)
    assert np.array_equal(Y.cpu().numpy().astype(np.int64), want)


def test_sharded_error_names_the_shard(alcop):
    """A failing shard (here: a schedule its shard cannot run) comes back on the
    caller's thread as "<RuleTag>: shard i: ..."."""
    M, N, K = 1024, 1024, 1024
    A = torch.zeros((M, K), device="cuda", dtype=torch.bfloat16)
    B = torch.zeros((K, N), device="cuda", dtype=torch.bfloat16)
    C = torch.zeros((M, N), device="cuda", dtype=torch.bfloat16)
    bad = alcop.make_schedule(tileN=256, tileK=128, n_stage=6)  # over the shared-memory budget
    shards = [(0, None, A[:512], B, C[:512]), (0, None, A[512:], B, C[512:])]
    with pytest.raises(alcop.AlcopError) as ei:
        alcop.gemm_sharded(alcop.gemm_desc(M, N, K), shards, bad, 256)
    assert ei.value.rule == "SmemCapacity" and "shard 0" in str(ei.value)
