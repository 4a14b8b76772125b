"""Seeded conv2d fuzz on the GPU: random shapes of every kernel class
alcop_conv2d routes to (stem pixel pairs, window with a resident or streamed
filter on one CTA or a CTA pair, 1x1 on the GEMM kernels, im2col on one CTA or
a pair, the small-channel im2col) x the chooser's pick and random schedules of
that class, with bf16 or fp16 inputs and fp32 / bf16 / fp16 outputs,
bit-exact against the oracle's direct convolution on the reference's integer
inputs (16-bit outputs compared as RNE bit patterns).  A random schedule may be rejected — then only
with a configuration error naming a rule tag, never a crash or wrong bits."""
import numpy as np
import pytest

from oracle import coracle
from oracle.splitmix import random_tensor

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

CLASSES = ("stem", "window", "stream", "gemm1x1", "im2col64", "im2col_small")
TAGS = ("SmemCapacity", "TmemCapacity", "BadSchedule", "BadTile", "BadStages", "Unsupported")


def _shape(rng, cls):
    """(N, H, W, C, K, R, S, stride, pad) of the class."""
    N = int(rng.integers(1, 4))
    if cls == "stem":
        R = int(rng.integers(1, 8))
        S = int(rng.integers(1, 8))
        W = 16 * int(rng.integers(1, 5))
        return (N, int(rng.integers(R, 40)), W, int(rng.choice([3, 4])), int(rng.choice([64, 128])), R, S,
                (int(rng.integers(1, 3)), 2), (int(rng.integers(0, R // 2 + 1)), int(rng.integers(0, S // 2 + 1))))
    if cls in ("window", "stream"):
        R, S = int(rng.integers(1, 4)), int(rng.integers(2, 4))
        H = int(rng.integers(max(R, 4), 40))
        W = int(rng.integers(max(S, 4), 60))
        C = 64 if cls == "window" else int(rng.choice([128, 192, 256]))
        K = int(rng.choice([64, 128])) if cls == "window" else int(rng.choice([32, 64, 96, 128]))
        return (N, H, W, C, K, R, S, (1, 1), (int(rng.integers(0, R)), int(rng.integers(0, S))))
    if cls == "gemm1x1":
        H, W = int(rng.integers(2, 30)), int(rng.integers(2, 30))
        return (N, H, W, int(rng.choice([64, 128, 256])), int(rng.choice([64, 128, 192, 256])), 1, 1, (1, 1),
                (0, 0))
    if cls == "im2col64":
        R = int(rng.integers(1, 4))
        st = int(rng.integers(1, 3))
        H = int(rng.integers(R + 2, 24))
        return (N, H, H, int(rng.choice([64, 128])), int(rng.choice([64, 128, 256])), R, R, (st, st),
                (int(rng.integers(0, R)),) * 2)
    R = int(rng.integers(1, 6))
    H = int(rng.integers(R + 2, 20))
    return (N, H, H, int(rng.choice([8, 16, 24, 40])), int(rng.choice([64, 128])), R, R, (1, 1),
            (int(rng.integers(0, R)),) * 2)


def _random_schedules(alcop, rng, cls, K, S):
    out = []
    for _ in range(2):
        if cls in ("stem", "window"):
            out.append(alcop.make_schedule(tileN=K, tileK=64, n_stage=int(rng.integers(1, 6)),
                                           n_stage_inner=int(rng.integers(1, 4)),
                                           cta_group=1 if cls == "stem" else int(rng.integers(1, 3))))
        elif cls == "stream":
            out.append(alcop.make_schedule(tileN=K, tileK=int(rng.choice([64, 64 * S])),
                                           n_stage=int(rng.integers(1, 4)), n_stage_B=int(rng.integers(1, 6)),
                                           n_stage_inner=int(rng.integers(1, 3)), cta_group=int(rng.integers(1, 3))))
        else:
            cg = int(rng.integers(1, 3)) if cls != "im2col_small" else 1
            tn = int(rng.choice([64, 128, 192, 256])) if cg == 1 else int(rng.choice([128, 192, 256]))
            out.append(alcop.make_schedule(tileN=tn, tileK=64, n_stage=int(rng.integers(1, 7)), cta_group=cg))
    return out


@pytest.mark.parametrize("seed", range(90))
def test_conv_fuzz(alcop, seed):
    rng = np.random.default_rng(1000 + seed)
    cls = CLASSES[seed % len(CLASSES)]
    N, H, W, C, K, R, S, st, pd = _shape(rng, cls)
    if (H + 2 * pd[0] - R) < 0 or (W + 2 * pd[1] - S) < 0:
        pytest.skip("empty output")
    in_dt = ("bf16", "f16")[int(rng.integers(0, 2))]
    out_dt = ("f32", "bf16", "f16")[int(rng.integers(0, 3))]
    tdt = {"bf16": torch.bfloat16, "f16": torch.float16, "f32": torch.float32}
    x = random_tensor(N * H * W * C, 500 + seed).reshape(N, H, W, C)
    w = random_tensor(K * R * S * C, 700 + seed).reshape(K, R, S, C)
    ref = coracle.conv2d(coracle.to_dtype(x.astype(np.float32), in_dt), coracle.to_dtype(w.astype(np.float32), in_dt),
                         st, pd, in_dt, out_dt)
    X = torch.from_numpy(x).to(tdt[in_dt]).cuda()
    Wt = torch.from_numpy(w).to(tdt[in_dt]).cuda()
    scheds = [None] + _random_schedules(alcop, rng, cls, K, S)
    ran = 0
    for s in scheds:
        try:
            Y = alcop.conv2d(X, Wt, st, pd, sched=s, out_dtype=tdt[out_dt])
        except alcop.AlcopError as e:
            assert s is not None and any(t in str(e) for t in TAGS), (cls, (N, H, W, C, K, R, S, st, pd), s, e)
            continue
        torch.cuda.synchronize()
        got = Y.cpu().numpy() if out_dt == "f32" else Y.cpu().view(torch.int16).numpy().view(np.uint16)
        if not np.array_equal(got, ref):
            bad = np.argwhere(got != ref)
            raise AssertionError("%s %s %s->%s %s: %d mismatches, first at %s: got %s want %s" % (
                cls, (N, H, W, C, K, R, S, st, pd), in_dt, out_dt, s, len(bad), bad[0].tolist(), got[tuple(bad[0])],
                ref[tuple(bad[0])]))
        ran += 1
    assert ran >= 1  # the chooser's pick always runs
