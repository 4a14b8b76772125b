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
    # small-channel path (8-channel im2col boxes, no-swizzle core matrices)
    (2, 30, 30, 3, 64, 7, 7, 2, 3),  # ResNet-50 conv1 shape class, C padded 3 -> 8
    (2, 10, 10, 8, 64, 3, 3, 1, 1),
    (1, 12, 12, 16, 128, 3, 3, 2, 1),
    (2, 9, 9, 24, 64, 5, 5, 1, 2),
    (1, 8, 8, 40, 192, 1, 1, 1, 0),
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
    """The C ABI itself rejects C % 8 != 0 (the Python wrapper pads NHWC channels first)."""
    import ctypes
    X = torch.zeros(1, 8, 8, 3, dtype=torch.bfloat16, device="cuda")
    Wt = torch.zeros(64, 7, 7, 3, dtype=torch.bfloat16, device="cuda")
    Y = torch.zeros(1, 4, 4, 64, dtype=torch.bfloat16, device="cuda")
    d = alcop.conv_desc(1, 8, 8, 3, 64, 7, 7, (2, 2), (3, 3), alcop.BF16, alcop.BF16)
    s = alcop.make_schedule(tileN=64, tileK=64, n_stage=2)
    lib = alcop.load_library()
    rc = lib.alcop_conv2d(ctypes.byref(d), ctypes.byref(s), ctypes.c_void_p(X.data_ptr()),
                          ctypes.c_void_p(Wt.data_ptr()), ctypes.c_void_p(Y.data_ptr()), None)
    assert rc == alcop.ALCOP_ERR_CONFIG
    assert lib.alcop_last_error().decode().startswith("Unsupported")


def test_conv1_small_channel_schedules(alcop):
    """conv1 class (7x7/2, C 3 -> 8) across tiles, stages and modes, bf16 out."""
    N, H, W, C, K = 2, 24, 24, 3, 64
    x = random_tensor(N * H * W * C, 41).reshape(N, H, W, C)
    w = random_tensor(K * 49 * C, 42).reshape(K, 7, 7, C)
    ref = coracle.conv2d(coracle.to_dtype(x.astype(np.float32), "bf16"),
                         coracle.to_dtype(w.astype(np.float32), "bf16"), (2, 2), (3, 3), "bf16", "f32")
    X = torch.from_numpy(x).to(torch.bfloat16).cuda()
    Wt = torch.from_numpy(w).to(torch.bfloat16).cuda()
    want = torch.from_numpy(ref).to(torch.bfloat16)
    for tn, st, mode in ((64, 2, 0), (64, 6, 1), (128, 4, 1), (64, 1, 1)):
        s = alcop.make_schedule(tileN=tn, tileK=64, n_stage=st, n_stage_inner=2 if st > 1 else 1, mode=mode)
        Y = alcop.conv2d(X, Wt, (2, 2), (3, 3), sched=s, out_dtype=torch.bfloat16)
        assert torch.equal(Y.cpu(), want), (tn, st, mode)


STEM_CASES = [  # N, H, W, C, K, R, S, stride, pad  (halo-padded input, S*C <= 64)
    (2, 30, 30, 3, 64, 7, 7, 2, 3),    # conv1 class, C 3 -> 8
    (1, 35, 37, 3, 64, 7, 7, 2, 3),    # ragged 8 x 16 output blocks
    (2, 20, 24, 8, 128, 3, 3, 1, 1),
    (1, 18, 18, 16, 64, 4, 4, 2, 1),
    (2, 12, 40, 8, 64, 5, 8, 1, 2),    # S*C = 64
    (1, 16, 16, 64, 64, 1, 1, 1, 0),
]


@pytest.mark.parametrize("case", STEM_CASES, ids=lambda c: "x".join(map(str, c)))
@pytest.mark.parametrize("out_dt", ["f32", "bf16"])
def test_conv_stem_halo_exact(alcop, case, out_dt):
    """Stem kernel (one TMA box per filter row over the halo-padded input)."""
    N, H, W, C, K, R, S, st, pd = case
    x = random_tensor(N * H * W * C, 51).reshape(N, H, W, C)
    w = random_tensor(K * R * S * C, 52).reshape(K, R, S, C)
    ref = coracle.conv2d(coracle.to_dtype(x.astype(np.float32), "bf16"),
                         coracle.to_dtype(w.astype(np.float32), "bf16"), (st, st), (pd, pd), "bf16", "f32")
    X = torch.from_numpy(x).to(torch.bfloat16).cuda()
    Xh = torch.nn.functional.pad(X, (0, 0, pd, pd, pd, pd))  # the halo layout [N, H+2p, W+2p, C]
    Wt = torch.from_numpy(w).to(torch.bfloat16).cuda()
    odt = torch.float32 if out_dt == "f32" else torch.bfloat16
    for tn, stg, mode in ((64, 4, 1), (128, 2, 0)):
        if tn > K:
            continue
        s = alcop.make_schedule(tileN=tn, tileK=64, n_stage=stg, n_stage_inner=2, mode=mode)
        Y = alcop.conv2d(Xh, Wt, (st, st), (pd, pd), sched=s, out_dtype=odt, x_halo=True)
        want = torch.from_numpy(ref).to(odt)
        got = Y.cpu()
        if not torch.equal(got, want):
            bad = torch.nonzero(got != want)
            raise AssertionError("mismatch (n=%d) at %s" % (len(bad), bad[:4].tolist()))


GEMM_CASES = [  # 1x1 / stride 1 / no padding: the conv runs on the GEMM kernels (CTA pairs included)
    (2, 14, 14, 256, 1024),
    (1, 7, 7, 512, 2048),
    (3, 9, 11, 64, 256),
]


@pytest.mark.parametrize("case", GEMM_CASES, ids=lambda c: "x".join(map(str, c)))
def test_conv_1x1_on_gemm_kernels(alcop, case):
    N, H, W, C, K = case
    x = random_tensor(N * H * W * C, 61).reshape(N, H, W, C)
    w = random_tensor(K * C, 62).reshape(K, 1, 1, C)
    ref = coracle.conv2d(coracle.to_dtype(x.astype(np.float32), "bf16"),
                         coracle.to_dtype(w.astype(np.float32), "bf16"), (1, 1), (0, 0), "bf16", "f32")
    X = torch.from_numpy(x).to(torch.bfloat16).cuda()
    Wt = torch.from_numpy(w).to(torch.bfloat16).cuda()
    want = torch.from_numpy(ref).to(torch.bfloat16)
    d = alcop.conv_desc(N, H, W, C, K, 1, 1, (1, 1), (0, 0), alcop.BF16, alcop.BF16)
    scheds = [alcop.choose_conv_schedule(d), alcop.make_schedule(tileN=256, tileK=64, n_stage=6, cta_group=2),
              alcop.make_schedule(tileN=128, tileK=64, n_stage=4)]
    for s in scheds:
        Y = alcop.conv2d(X, Wt, (1, 1), (0, 0), sched=s, out_dtype=torch.bfloat16)
        assert torch.equal(Y.cpu(), want), s


PAIR_CASES = [  # N, H, W, C, K, R, S, stride, pad: implicit-GEMM conv on CTA pairs (C % 64 == 0)
    (2, 14, 14, 64, 256, 3, 3, 1, 1),
    (2, 16, 16, 128, 256, 3, 3, 2, 1),
    (2, 14, 14, 256, 512, 1, 1, 2, 0),   # strided 1x1 (downsample)
    (1, 9, 11, 64, 128, 3, 3, 1, 1),     # ragged: the last pair tile's second CTA past M
    (3, 7, 7, 128, 192, 3, 3, 1, 1),
]


@pytest.mark.parametrize("case", PAIR_CASES, ids=lambda c: "x".join(map(str, c)))
def test_conv_cta_pair_exact(alcop, case):
    N, H, W, C, K, R, S, st, pd = case
    x = random_tensor(N * H * W * C, 71).reshape(N, H, W, C)
    w = random_tensor(K * R * S * C, 72).reshape(K, R, S, C)
    ref = coracle.conv2d(coracle.to_dtype(x.astype(np.float32), "bf16"),
                         coracle.to_dtype(w.astype(np.float32), "bf16"), (st, st), (pd, pd), "bf16", "f32")
    X = torch.from_numpy(x).to(torch.bfloat16).cuda()
    Wt = torch.from_numpy(w).to(torch.bfloat16).cuda()
    ran = 0
    for tn, stg in ((256, 6), (128, 4), (192, 5)):
        if tn > K and tn != 128:
            continue
        s = alcop.make_schedule(tileN=tn, tileK=64, n_stage=stg, cta_group=2)
        for odt in (torch.float32, torch.bfloat16):
            Y = alcop.conv2d(X, Wt, (st, st), (pd, pd), sched=s, out_dtype=odt)
            assert torch.equal(Y.cpu(), torch.from_numpy(ref).to(odt)), (s, odt)
            ran += 1
    assert ran >= 2
