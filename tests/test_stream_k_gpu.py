"""GPU parity of the stream-K CTA-pair schedule (alcop_schedule.stream_k = 1).

The tiles' chunk stream is split evenly over the clusters; a tile cut between
two clusters is finished by the earlier one from the later one's fp32
partial.  D-int inputs: every partial and their sum are exact integers, so
the result must equal the exact product bit-for-bit (the same bar as the
whole-tile kernel), including bf16 output (RNE of the exact sum), ragged
M/N/K, batches, short K and repeated launches (the hand-off flags re-arm).
"""
import numpy as np
import pytest

from oracle.splitmix import gemm_inputs, uniform_tensor

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(autouse=True)
def _stream_k_workspace(alcop):
    """The caller-owned stream-K workspace (the library never allocates it)."""
    ws = alcop.set_stream_k_workspace(256 << 20)
    yield ws
    alcop.load_library().alcop_set_stream_k_workspace(None, 0)


def _sk(alcop, tileN=256, tileK=64, n_stage=6, stream_k=1):
    return alcop.make_schedule(tileN=tileN, tileK=tileK, n_stage=n_stage, cta_group=2, stream_k=stream_k)


def _check(alcop, M, N, K, batch=1, out_dt=torch.float32, in_dt=torch.bfloat16, sched=None, seed=0, reps=1):
    a, b = gemm_inputs(M, N, K, batch, seed=seed)
    # float64 BLAS product: exact for D-int inputs (|sum| <= 64 K << 2^53), far faster than an int64 matmul
    exact = np.rint(np.matmul(a.astype(np.float64), b.astype(np.float64))).astype(np.int64)
    A = torch.from_numpy(a).to(in_dt).cuda()
    B = torch.from_numpy(b).to(in_dt).cuda()
    ref = torch.from_numpy(exact.astype(np.float64)).to(torch.float32)
    if out_dt != torch.float32:
        ref = ref.to(out_dt)
    for r in range(reps):
        C = alcop.matmul(A, B, sched, out_dtype=out_dt)
        torch.cuda.synchronize()
        C = C.cpu()
        if not torch.equal(C, ref):
            d = (C.float() - ref.float()).abs()
            idx = torch.nonzero(d)[:5].tolist()
            raise AssertionError("rep %d: %d mismatches, first at %s" % (r, int((d != 0).sum()), idx))


@pytest.mark.parametrize("out", ["f32", "bf16"])
def test_stream_k_ffn1_exact(alcop, out):
    """FFN1 4096x3072x768 (192 pair tiles on 74 clusters: 31.1 chunks each)."""
    _check(alcop, 4096, 3072, 768, out_dt=torch.float32 if out == "f32" else torch.bfloat16, sched=_sk(alcop),
           seed=3)


@pytest.mark.parametrize("M,N,K,batch,tileN,tileK,st", [
    (4096, 2304, 128, 1, 256, 64, 6),   # short K: 2 chunks per tile
    (4000, 2000, 1000, 1, 256, 64, 6),  # ragged M, N and K
    (1024, 1024, 512, 5, 256, 64, 6),   # batch: 80 tiles
    (4096, 3072, 768, 1, 192, 64, 6),   # 96-column halves (padded B atoms)
    (4096, 1536, 1024, 1, 128, 128, 4),  # BK 128 (atom-view A)
    (2560, 2816, 640, 1, 256, 32, 8),   # BK 32
])
def test_stream_k_shapes_exact(alcop, M, N, K, batch, tileN, tileK, st):
    _check(alcop, M, N, K, batch=batch, sched=_sk(alcop, tileN=tileN, tileK=tileK, n_stage=st), seed=M + K)


def test_stream_k_repeated_launches_exact(alcop):
    """Back-to-back launches reuse the workspace: the finishers re-arm the flags."""
    _check(alcop, 4096, 3072, 768, out_dt=torch.bfloat16, sched=_sk(alcop), seed=9, reps=4)


def test_stream_k_fp16_exact(alcop):
    _check(alcop, 2048, 4096, 512, in_dt=torch.float16, out_dt=torch.float16, sched=_sk(alcop), seed=21)


def test_stream_k_float_inputs_close(alcop):
    """D-float: the split changes the fp32 summation order only (tolerance of SURVEY §8d)."""
    M, N, K = 4096, 3072, 768
    a = uniform_tensor(M * K, 5).reshape(M, K)
    b = uniform_tensor(K * N, 6).reshape(K, N)
    A = torch.from_numpy(a).to(torch.bfloat16).cuda()
    B = torch.from_numpy(b).to(torch.bfloat16).cuda()
    C = alcop.matmul(A, B, _sk(alcop), out_dtype=torch.float32)
    ref = A.double() @ B.double()
    rel = float((C.double() - ref).norm() / ref.norm())
    assert rel <= 1e-5, rel


def test_stream_k_rejected_outside_pairs(alcop):
    d = alcop.gemm_desc(1024, 1024, 512)
    with pytest.raises(alcop.AlcopError):
        alcop.validate(d, alcop.make_schedule(tileN=256, cta_group=1, stream_k=1))
    with pytest.raises(alcop.AlcopError):
        alcop.validate(d, alcop.make_schedule(tileN=256, cta_group=2, stream_k=1, mode=alcop.MODE_WRAP))


def test_stream_k_without_workspace_runs_whole_tiles(alcop):
    """No registered workspace (or one too small): the stream_k schedule runs
    whole tiles — still exact, and nothing is allocated on the call path."""
    lib = alcop.load_library()
    lib.alcop_set_stream_k_workspace(None, 0)
    _check(alcop, 4096, 3072, 768, sched=_sk(alcop), seed=9)
    small = torch.empty(8192, dtype=torch.uint8, device="cuda")
    assert lib.alcop_set_stream_k_workspace(small.data_ptr(), 8192) == 0
    d = alcop.gemm_desc(4096, 3072, 768)
    assert lib.alcop_stream_k_workspace_bytes(d, _sk(alcop)) > 8192
    _check(alcop, 4096, 3072, 768, sched=_sk(alcop), seed=10)
