"""GPU parity of the implicit-GEMM conv2d (K3, TMA im2col) against the
oracle's direct convolution (oracle/alcop_oracle.c §4), bit-exact on the
reference's integer inputs (fp32 accumulation of small integers is exact)."""
import numpy as np
import pytest

from oracle import coracle
from oracle.splitmix import random_tensor

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

CASES = [  # N, H, W, C, K, R, S, stride, pad
    (2, 8, 8, 64, 64, 1, 1, 1, 0),
    (2, 14, 14, 64, 128, 3, 3, 1, 1),
    (1, 16, 16, 128, 64, 3, 3, 2, 1),
    (3, 9, 11, 64, 192, 3, 3, 1, 1),
    (2, 14, 14, 128, 256, 1, 1, 2, 0),
    (1, 7, 7, 64, 64, 3, 3, 1, 1),
    (2, 12, 12, 64, 64, 5, 5, 1, 2),
    (1, 15, 15, 64, 128, 3, 3, 2, 0),
]


@pytest.mark.parametrize("case", CASES, ids=lambda c: "x".join(map(str, c)))
def test_conv_exact(alcop, case):
    N, H, W, C, K, R, S, st, pd = case
    x = random_tensor(N * H * W * C, 21).reshape(N, H, W, C)
    w = random_tensor(K * R * S * C, 22).reshape(K, R, S, C)
    xb = coracle.to_dtype(x.astype(np.float32), "bf16")
    wb = coracle.to_dtype(w.astype(np.float32), "bf16")
    ref = coracle.conv2d(xb, wb, (st, st), (pd, pd), "bf16", "f32")
    X = torch.from_numpy(x).to(torch.bfloat16).cuda()
    Wt = torch.from_numpy(w).to(torch.bfloat16).cuda()
    Y = alcop.conv2d(X, Wt, (st, st), (pd, pd), out_dtype=torch.float32)
    torch.cuda.synchronize()
    got = Y.cpu().numpy()
    assert got.shape == ref.shape
    if not np.array_equal(got, ref):
        bad = np.argwhere(got != ref)
        raise AssertionError("mismatch at %s (n=%d): got %s want %s" % (bad[:4].tolist(), len(bad),
                             got[tuple(bad[0])], ref[tuple(bad[0])]))


def test_conv_bf16_out_and_schedules(alcop):
    N, H, W, C, K = 2, 14, 14, 64, 128
    x = random_tensor(N * H * W * C, 31).reshape(N, H, W, C)
    w = random_tensor(K * 9 * C, 32).reshape(K, 3, 3, C)
    ref = coracle.conv2d(coracle.to_dtype(x.astype(np.float32), "bf16"),
                         coracle.to_dtype(w.astype(np.float32), "bf16"), (1, 1), (1, 1), "bf16", "f32")
    X = torch.from_numpy(x).to(torch.bfloat16).cuda()
    Wt = torch.from_numpy(w).to(torch.bfloat16).cuda()
    for tn, st, mode in ((64, 2, 0), (128, 4, 1), (256, 3, 0), (128, 1, 1)):
        s = alcop.make_schedule(tileN=tn, tileK=64, n_stage=st, n_stage_inner=2 if st > 1 else 1, mode=mode)
        Y = alcop.conv2d(X, Wt, (1, 1), (1, 1), sched=s, out_dtype=torch.bfloat16)
        want = torch.from_numpy(ref).to(torch.bfloat16)
        assert torch.equal(Y.cpu(), want), (tn, st, mode)


def test_conv_rejects_unsupported(alcop):
    X = torch.zeros(1, 8, 8, 3, dtype=torch.bfloat16, device="cuda")
    Wt = torch.zeros(64, 7, 7, 3, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(alcop.AlcopError) as ei:
        alcop.conv2d(X, Wt, (2, 2), (3, 3), sched=alcop.make_schedule(tileN=64, tileK=64, n_stage=2))
    assert ei.value.rule == "Unsupported"
