"""The oracle's sampled exact checkers (alcop_oracle.c §4b, used by the
scale-parity GPU tests) agree with its whole-problem int64 GEMM and direct
convolution, and its int8 generator draws the reference's SplitMix64 values."""
import numpy as np
import pytest

from oracle import coracle
from oracle.splitmix import random_tensor


def test_random_i8_is_random_tensor():
    for seed in (0, 1, 21, 1000003):
        assert np.array_equal(coracle.random_i8(5000, seed).astype(np.int64), random_tensor(5000, seed))


@pytest.mark.parametrize("batch,M,N,K", [(1, 70, 300, 96), (3, 33, 65, 40), (1, 5, 2500, 17)])
@pytest.mark.parametrize("b_layout", [0, 1])
def test_gemm_rows_cols_match_full(batch, M, N, K, b_layout):
    a = coracle.random_i8(batch * M * K, 0).reshape(batch, M, K)
    b = coracle.random_i8(batch * K * N, 1).reshape(batch, K, N)
    full = coracle.gemm_i64(a.astype(np.int64), b.astype(np.int64)).reshape(batch * M, N)
    bl = b if b_layout == 0 else np.ascontiguousarray(np.swapaxes(b, -1, -2))
    if batch == 1:
        a, bl = a[0], bl[0]
    rows = np.array([0, 1, batch * M - 1, (batch * M) // 2])
    cols = np.array([0, N - 1, N // 3])
    assert np.array_equal(coracle.gemm_rows_i8(a, bl, rows, b_layout), full[rows])
    assert np.array_equal(coracle.gemm_cols_i8(a, bl, cols, b_layout), full[:, cols])


@pytest.mark.parametrize("case", [(2, 9, 9, 3, 16, 7, 7, 2, 3), (1, 8, 8, 16, 8, 3, 3, 1, 1),
                                  (2, 10, 10, 8, 4, 1, 1, 2, 0), (1, 11, 11, 24, 8, 3, 3, 2, 1)])
def test_conv_points_match_direct_conv(case):
    N, H, W, C, K, R, S, st, pd = case
    x = coracle.random_i8(N * H * W * C, 21).reshape(N, H, W, C)
    w = coracle.random_i8(K * R * S * C, 22).reshape(K, R, S, C)
    full = coracle.conv2d(coracle.to_dtype(x.astype(np.float32), "f32"), coracle.to_dtype(w.astype(np.float32), "f32"),
                          (st, st), (pd, pd), "f32", "f32")
    P, Q = full.shape[1:3]
    pts = np.array([(n, p, q) for n in range(N) for p in range(P) for q in range(Q)], dtype=np.int64)
    got = coracle.conv2d_points_i8(x, w, (st, st), (pd, pd), pts)
    assert np.array_equal(got, full.reshape(-1, K).astype(np.int64))
