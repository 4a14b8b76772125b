"""Exact parity at the sizes bench.py times, with the
schedules the bench runs.

The reference checks every transformed program against the untransformed
one (cli.hpp:285-304 -> check_equivalence, interp.hpp:469-509).  Here the
checker is the oracle's exact integer product on the reference's D-int inputs
(SplitMix64 range(-8,8), cli.hpp:41-46): exact in bf16, every fp32 partial sum
an integer below 2^24, so the kernel's bf16 output must equal the
round-to-nearest-even of the exact integer result bit for bit.

* C2 BERT-layer GEMMs and C3 attention BMMs (batch 192): the whole output.
* C5 squares 4096..16384: one full row in every 256-row tile row and one full
  column in every 256-column tile column (plus the first/last row/column), so
  every output tile is checked along one row and one column.
* C4 ResNet-50 layers at batch 256 (conv1 stem on the NHWC8 halo-padded
  input included): 2048 output pixels x all K channels per layer, including
  every corner pixel of the first and last image.
"""
import zlib

import numpy as np
import pytest

from oracle import coracle
from paper_2210_16691_b200 import workloads as W

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _dev_bf16(a_i8):
    return torch.from_numpy(a_i8).cuda().to(torch.bfloat16)


def _rne_bf16(exact_i64):
    """exact integer -> fp32 (exact, |v| < 2^24) -> bf16 RNE, as float32 values."""
    bits = coracle.to_dtype(exact_i64.astype(np.float32), "bf16")
    return coracle.to_f32(bits, "bf16")


def _compare(got_f32, exact_i64, what):
    want = _rne_bf16(exact_i64)
    if not np.array_equal(got_f32, want):
        bad = np.argwhere(got_f32 != want)
        raise AssertionError("%s: %d mismatches, first at %s: got %s want %s (exact %s)" % (
            what, len(bad), bad[0].tolist(), got_f32[tuple(bad[0])], want[tuple(bad[0])], exact_i64[tuple(bad[0])]))


def _tile_samples(n, tile, rng):
    """One index inside every tile of `tile` along a dimension of size n, plus both ends."""
    idx = [min(n - 1, t + int(rng.integers(0, tile))) for t in range(0, n, tile)]
    return np.array(sorted(set(idx + [0, n - 1])), dtype=np.int64)


# ------------------------------------------------------------------ C5
@pytest.mark.parametrize("n", W.SQUARES)
def test_square_sampled_exact(alcop, n):
    a = coracle.random_i8(n * n, 0).reshape(n, n)
    b = coracle.random_i8(n * n, 1).reshape(n, n)
    s = W.square_schedule(alcop, n, n)
    C = alcop.matmul(_dev_bf16(a), _dev_bf16(b), s, out_dtype=torch.bfloat16)
    torch.cuda.synchronize()
    rng = np.random.default_rng(n)
    rows = _tile_samples(n, W.SQUARE_GRANULE, rng)
    cols = _tile_samples(n, 256, rng)
    got_rows = C[torch.from_numpy(rows).cuda()].float().cpu().numpy()
    got_cols = C[:, torch.from_numpy(cols).cuda()].float().cpu().numpy()
    _compare(got_rows, coracle.gemm_rows_i8(a, b, rows), "square %d rows (%s)" % (n, s))
    _compare(got_cols, coracle.gemm_cols_i8(a, b, cols), "square %d cols (%s)" % (n, s))


@pytest.mark.parametrize("world", [2, 8])
def test_square_m_shard_exact(alcop, world):
    """Every rank's shard of the M-sharded 16384^3 problem (rows of A/C in
    256-row granules, B replicated) computed with that shard's own schedule
    equals the same rows of the exact product."""
    from paper_2210_16691_b200.sharded import all_shards
    n = 16384
    a = coracle.random_i8(n * n, 0).reshape(n, n)
    b = coracle.random_i8(n * n, 1).reshape(n, n)
    B = _dev_bf16(b)
    rng = np.random.default_rng(world)
    for sh in all_shards(n, world, granule=W.SQUARE_GRANULE):
        m = sh.size
        s = W.square_schedule(alcop, m, n)
        C = alcop.matmul(_dev_bf16(np.ascontiguousarray(a[sh.start:sh.stop])), B, s, out_dtype=torch.bfloat16)
        torch.cuda.synchronize()
        rows = _tile_samples(m, 128, rng)
        got = C[torch.from_numpy(rows).cuda()].float().cpu().numpy()
        _compare(got, coracle.gemm_rows_i8(a, b, rows + sh.start), "shard %d/%d rows" % (sh.rank, world))
        del C


# ------------------------------------------------------------------ C3
@pytest.mark.parametrize("name,M,N,K", W.BMM_ATTENTION, ids=[g[0] for g in W.BMM_ATTENTION])
def test_bmm_attention_b192_exact(alcop, name, M, N, K):
    bt = W.BMM_BATCH
    a = coracle.random_i8(bt * M * K, 0).reshape(bt, M, K)
    b = coracle.random_i8(bt * K * N, 1).reshape(bt, K, N)
    exact = coracle.gemm_rows_i8(a, b, np.arange(bt * M)).reshape(bt, M, N)
    A, B = _dev_bf16(a), _dev_bf16(b)
    C = torch.empty((bt, M, N), dtype=torch.bfloat16, device="cuda")
    tuned, trials = alcop.tune(A, B, C, budget=8)
    model = alcop.choose_schedule(alcop.gemm_desc(M, N, K, bt, alcop.BF16, alcop.BF16, alcop.B_KN))
    for label, s in (("model", model), ("tuned", tuned)):
        C.zero_()
        alcop.matmul(A, B, s, out=C)
        torch.cuda.synchronize()
        _compare(C.float().cpu().numpy(), exact, "%s %s (%s)" % (name, label, s))
    # the n_stage = 1 variant the bench times beside it
    s1 = alcop.make_schedule(tileN=tuned.tileN, tileK=tuned.tileK, n_stage=1, n_stage_inner=1)
    alcop.matmul(A, B, s1, out=C)
    torch.cuda.synchronize()
    _compare(C.float().cpu().numpy(), exact, "%s n_stage=1" % name)


# ------------------------------------------------------------------ C2
@pytest.mark.parametrize("name,M,N,K", W.BERT_GEMMS, ids=[g[0] for g in W.BERT_GEMMS])
def test_bert_layer_gemm_exact(alcop, name, M, N, K):
    a = coracle.random_i8(M * K, 0).reshape(M, K)
    b = coracle.random_i8(K * N, 1).reshape(K, N)
    exact = coracle.gemm_rows_i8(a, b, np.arange(M))
    A, B = _dev_bf16(a), _dev_bf16(b)
    C = torch.empty((M, N), dtype=torch.bfloat16, device="cuda")
    tuned, _ = alcop.tune(A, B, C, budget=8)
    model = alcop.choose_schedule(alcop.gemm_desc(M, N, K, 1, alcop.BF16, alcop.BF16, alcop.B_KN))
    for label, s in (("model", model), ("tuned", tuned)):
        C.zero_()
        alcop.matmul(A, B, s, out=C)
        torch.cuda.synchronize()
        _compare(C.float().cpu().numpy(), exact, "%s %s (%s)" % (name, label, s))


# ------------------------------------------------------------------ C4
def _conv_points(nimg, P, rng, count=2048):
    corners = [(n, p, q) for n in (0, nimg - 1) for p in (0, P - 1) for q in (0, P - 1)]
    rand = np.stack([rng.integers(0, nimg, count), rng.integers(0, P, count), rng.integers(0, P, count)], 1)
    return np.concatenate([np.array(corners, dtype=np.int64), rand.astype(np.int64)])


@pytest.mark.parametrize("layer", W.CONV_LAYERS, ids=[c.name for c in W.CONV_LAYERS])
def test_resnet50_conv_b256_sampled_exact(alcop, layer):
    nimg = W.RESNET_BATCH
    L = layer
    x = coracle.random_i8(nimg * L.H * L.H * L.C, 21).reshape(nimg, L.H, L.H, L.C)
    w = coracle.random_i8(L.K * L.R * L.R * L.C, 22).reshape(L.K, L.R, L.R, L.C)
    hp = L.pad if L.halo else 0
    X = torch.zeros((nimg, L.H + 2 * hp, L.H + 2 * hp, L.Cs), dtype=torch.bfloat16, device="cuda")
    X[:, hp:hp + L.H, hp:hp + L.H, :L.C] = _dev_bf16(x)
    Wf = torch.zeros((L.K, L.R, L.R, L.Cs), dtype=torch.bfloat16, device="cuda")
    Wf[..., :L.C] = _dev_bf16(w)
    s = W.conv_schedule(alcop, L, nimg)
    Y = alcop.conv2d(X, Wf, (L.stride, L.stride), (L.pad, L.pad), sched=s, out_dtype=torch.bfloat16,
                     x_halo=L.halo)
    torch.cuda.synchronize()
    assert tuple(Y.shape) == (nimg, L.P, L.P, L.K)
    pts = _conv_points(nimg, L.P, np.random.default_rng(zlib.crc32(L.name.encode())))
    pt = torch.from_numpy(pts).cuda()
    got = Y[pt[:, 0], pt[:, 1], pt[:, 2]].float().cpu().numpy()
    exact = coracle.conv2d_points_i8(x, w, (L.stride, L.stride), (L.pad, L.pad), pts)
    _compare(got, exact, "%s (%s)" % (L.name, s))
