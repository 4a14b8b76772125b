"""GPU parity of the stem kernel (csrc/stem_sm100.cu: C = 4, horizontal stride
2, the A operand read straight from the raw input rows through overlapping
no-swizzle descriptors) against the oracle's direct convolution, bit-exact on
the reference's integer inputs.  ResNet-50 conv1 (7x7/2, 3 -> 64) is the
shape class; the cases also cover odd/even padding and filter widths, more
than one 128-column block per output row, stride_h 1, K = 128/256, and every
ring depth / accumulator count the space holds."""
import ctypes

import numpy as np
import pytest

from oracle import coracle
from oracle.splitmix import random_tensor

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

CASES = [  # N, H, W, C, K, R, S, (stride_h, stride_w), (pad_h, pad_w)
    (2, 32, 32, 3, 64, 7, 7, (2, 2), (3, 3)),     # conv1 class (C 3 -> 4)
    (1, 224, 224, 3, 64, 7, 7, (2, 2), (3, 3)),   # conv1, one whole image
    (1, 22, 288, 4, 128, 5, 5, (2, 2), (2, 2)),   # Q = 144: two column blocks; even pad
    (2, 17, 48, 4, 64, 4, 4, (1, 2), (0, 0)),     # stride_h 1, even S, no padding
    (1, 9, 64, 4, 256, 3, 3, (2, 2), (1, 1)),     # K = 256
    (2, 12, 16, 2, 64, 1, 1, (2, 2), (0, 0)),     # 1x1 / 2 (one tap, zero partner)
    (1, 20, 32, 3, 64, 6, 3, (3, 2), (2, 1)),     # stride_h 3, R != S
    (1, 5, 32, 3, 64, 7, 7, (2, 2), (3, 3)),      # image shorter than the filter (window box > H)
    (1, 9, 48, 3, 64, 7, 7, (2, 2), (3, 3)),      # stem, 5 output rows: a ragged four-row tile
    (3, 14, 32, 4, 64, 7, 7, (2, 2), (3, 3)),     # stem, 7 output rows, several images per CTA
]


def _inputs(case, seed):
    N, H, W, C, K, R, S, st, pd = case
    x = random_tensor(N * H * W * C, seed).reshape(N, H, W, C)
    w = random_tensor(K * R * S * C, seed + 1).reshape(K, R, S, C)
    ref = coracle.conv2d(coracle.to_dtype(x.astype(np.float32), "bf16"),
                         coracle.to_dtype(w.astype(np.float32), "bf16"), st, pd, "bf16", "f32")
    return (torch.from_numpy(x).to(torch.bfloat16).cuda(), torch.from_numpy(w).to(torch.bfloat16).cuda(), ref)


def _assert_equal(got, want, what):
    if not torch.equal(got, want):
        bad = torch.nonzero(got != want)
        raise AssertionError("%s: mismatch (n=%d) at %s: got %s want %s" % (
            what, len(bad), bad[:4].tolist(), got[tuple(bad[0])].item(), want[tuple(bad[0])].item()))


@pytest.mark.parametrize("case", CASES, ids=lambda c: "x".join(map(str, c[:7])) + "_s%d%d_p%d%d" % (*c[7], *c[8]))
@pytest.mark.parametrize("out_dt", ["f32", "bf16"])
def test_stem_exact(alcop, case, out_dt):
    X, Wt, ref = _inputs(case, 61)
    _, _, _, _, K, _, _, st, pd = case
    odt = torch.float32 if out_dt == "f32" else torch.bfloat16
    d = alcop.conv_desc(*case[:7], st, pd, alcop.BF16, alcop.F32 if out_dt == "f32" else alcop.BF16)
    d.C = 4
    s = alcop.choose_conv_schedule(d)
    assert s.tileN == K and s.cta_group == 1
    Y = alcop.conv2d(X, Wt, st, pd, out_dtype=odt)
    torch.cuda.synchronize()
    _assert_equal(Y.cpu(), torch.from_numpy(ref).to(odt), "model schedule %s" % s)


@pytest.mark.parametrize("case", [(2, 30, 64, 3, 64, 7, 7, (2, 2), (3, 3)),    # the stem: four-row tiles
                                  (2, 30, 64, 3, 64, 7, 7, (2, 2), (2, 3))],   # pad_h 2: one-row tiles
                         ids=["stem4", "pairs"])
def test_stem_schedules(alcop, case):
    """Every ring depth 1..8 x accumulators 1..4 that fits: same bits."""
    X, Wt, ref = _inputs(case, 71)
    want = torch.from_numpy(ref).to(torch.bfloat16)
    ran = 0
    for st in (1, 2, 3, 5, 8):
        for inner in (1, 2, 4):
            s = alcop.make_schedule(tileN=64, tileK=64, n_stage=st, n_stage_inner=inner, mode=1)
            try:
                Y = alcop.conv2d(X, Wt, case[7], case[8], sched=s, out_dtype=torch.bfloat16)
            except alcop.AlcopError as e:  # a ring / accumulator ring that does not fit this mode
                assert "SmemCapacity" in str(e) or "TmemCapacity" in str(e), e
                continue
            ran += 1
            _assert_equal(Y.cpu(), want, "stages %d inner %d" % (st, inner))
    assert ran >= 8


def test_stem_fourth_channel_and_grid(alcop):
    """A genuine 4-channel input (no zero channel) and a small persistent grid
    (each CTA walks many tiles through the rings)."""
    case = (3, 40, 96, 4, 64, 7, 7, (2, 2), (3, 3))
    X, Wt, ref = _inputs(case, 81)
    s = alcop.make_schedule(tileN=64, tileK=64, n_stage=3, n_stage_inner=2, mode=1)
    s.num_ctas = 5
    Y = alcop.conv2d(X, Wt, (2, 2), (3, 3), sched=s, out_dtype=torch.float32)
    _assert_equal(Y.cpu(), torch.from_numpy(ref), "grid 5")


def test_stem_float_inputs(alcop):
    """Float inputs: fp32 accumulation against a float64 direct conv (torch)."""
    g = torch.Generator().manual_seed(5)
    x = torch.rand(2, 64, 64, 3, generator=g) * 2 - 1
    w = torch.rand(64, 7, 7, 3, generator=g) * 2 - 1
    xb, wb = x.to(torch.bfloat16), w.to(torch.bfloat16)
    ref = torch.nn.functional.conv2d(xb.double().permute(0, 3, 1, 2), wb.double().permute(0, 3, 1, 2),
                                     stride=2, padding=3).permute(0, 2, 3, 1)
    Y = alcop.conv2d(xb.cuda(), wb.cuda(), (2, 2), (3, 3), out_dtype=torch.float32).cpu().double()
    err = (Y - ref).norm() / ref.norm()
    assert err < 1e-5, err


def test_stem_rejects(alcop):
    """The ABI's C = 4 path names what it cannot run (and never falls back)."""
    lib = alcop.load_library()
    X = torch.zeros(1, 16, 40, 4, dtype=torch.bfloat16, device="cuda")
    Wt = torch.zeros(64, 7, 7, 4, dtype=torch.bfloat16, device="cuda")
    Y = torch.zeros(1, 8, 20, 64, dtype=torch.bfloat16, device="cuda")

    def call(d, s):
        return lib.alcop_conv2d(ctypes.byref(d), ctypes.byref(s), ctypes.c_void_p(X.data_ptr()),
                                ctypes.c_void_p(Wt.data_ptr()), ctypes.c_void_p(Y.data_ptr()), None)

    good = alcop.make_schedule(tileN=64, tileK=64, n_stage=2, n_stage_inner=2, mode=1)
    d = alcop.conv_desc(1, 16, 40, 4, 64, 7, 7, (2, 2), (3, 3), alcop.BF16, alcop.BF16)  # W % 16 != 0
    assert call(d, good) == alcop.ALCOP_ERR_CONFIG
    assert lib.alcop_last_error().decode().startswith("Unsupported")
    d = alcop.conv_desc(1, 16, 32, 4, 64, 7, 7, (2, 2), (3, 3), alcop.BF16, alcop.BF16)
    for bad, tag in ((dict(tileN=128), "BadSchedule"), (dict(mode=0), "BadSchedule"),
                     (dict(n_stage_inner=4), "TmemCapacity"),  # the stem's four-row accumulators: 256 columns
                     (dict(n_stage_inner=2, tileN=64), None)):
        s = alcop.make_schedule(**{**dict(tileN=64, tileK=64, n_stage=2, n_stage_inner=2, mode=1), **bad})
        rc = call(d, s)
        if tag is None:
            assert rc == 0, lib.alcop_last_error()
        else:
            assert rc == alcop.ALCOP_ERR_CONFIG and lib.alcop_last_error().decode().startswith(tag), bad
    torch.cuda.synchronize()


# ----------------------------------------------------------------------------
# Window mode (C = 64, stride 1): a tile of TR output rows loads its input
# window once; tap (r, s) = the window shifted by r rows and s pixels, read
# through a 128B-swizzled descriptor whose start moved by whole 128-byte rows.
WINDOW_CASES = [  # N, H, W, C, K, R, S, (stride), (pad)
    (2, 56, 56, 64, 64, 3, 3, (1, 1), (1, 1)),    # ResNet-50 l1 3x3 class: pitch 64, 2 rows per tile
    (2, 28, 28, 64, 64, 3, 3, (1, 1), (1, 1)),    # pitch 32, 4 rows
    (2, 14, 14, 64, 64, 3, 3, (1, 1), (1, 1)),    # pitch 16, 8 rows (two output rows per epilogue warp)
    (1, 30, 30, 64, 64, 3, 3, (1, 1), (1, 1)),    # ragged last row block
    (2, 18, 18, 64, 64, 3, 3, (1, 1), (0, 0)),    # no padding
    (1, 9, 60, 64, 128, 1, 3, (1, 1), (0, 1)),    # R != S, K = 128
    (1, 12, 20, 64, 64, 2, 4, (1, 1), (1, 2)),    # even filter, uneven padding
    (1, 8, 8, 64, 64, 3, 3, (1, 1), (1, 1)),      # window box (10 rows) taller than the image
]


@pytest.mark.parametrize("case", WINDOW_CASES, ids=lambda c: "x".join(map(str, c[:7])) + "_p%d%d" % c[8])
@pytest.mark.parametrize("out_dt", ["f32", "bf16"])
def test_window_exact(alcop, case, out_dt):
    X, Wt, ref = _inputs(case, 91)
    _, _, _, _, K, _, _, st, pd = case
    odt = torch.float32 if out_dt == "f32" else torch.bfloat16
    d = alcop.conv_desc(*case[:7], st, pd, alcop.BF16, alcop.F32 if out_dt == "f32" else alcop.BF16)
    s = alcop.choose_conv_schedule(d)
    assert s.tileN == K, s  # the resident-filter (window) space
    Y = alcop.conv2d(X, Wt, st, pd, sched=s, out_dtype=odt)
    torch.cuda.synchronize()
    _assert_equal(Y.cpu(), torch.from_numpy(ref).to(odt), "window %s" % s)


def test_window_schedules_and_im2col_agree(alcop):
    """Every ring depth x accumulator count of the window mode, and the im2col
    kernel on the same conv (a WRAP schedule routes there): same bits."""
    case = (2, 56, 56, 64, 64, 3, 3, (1, 1), (1, 1))
    X, Wt, ref = _inputs(case, 93)
    want = torch.from_numpy(ref).to(torch.bfloat16)
    for st in (1, 2, 3):
        for inner in (1, 2, 4):
            s = alcop.make_schedule(tileN=64, tileK=64, n_stage=st, n_stage_inner=inner, mode=1)
            Y = alcop.conv2d(X, Wt, (1, 1), (1, 1), sched=s, out_dtype=torch.bfloat16)
            _assert_equal(Y.cpu(), want, "window stages %d inner %d" % (st, inner))
    s = alcop.make_schedule(tileN=64, tileK=64, n_stage=4, n_stage_inner=2, mode=0)  # WRAP: im2col kernel
    Y = alcop.conv2d(X, Wt, (1, 1), (1, 1), sched=s, out_dtype=torch.bfloat16)
    _assert_equal(Y.cpu(), want, "im2col")


# ----------------------------------------------------------------------------
# Window mode with a streamed filter (C = 64 x CB, stride 1): per channel block
# the window is one chunk of the A ring, the filter comes in chunks of TB taps
# (tileK = 64 x TB) through the B ring — separate A / B stage counts.
STREAM_CASES = [  # N, H, W, C, K, R, S, (stride), (pad)
    (2, 28, 28, 128, 128, 3, 3, (1, 1), (1, 1)),   # ResNet-50 l2 3x3 class
    (1, 14, 14, 256, 128, 3, 3, (1, 1), (1, 1)),   # four channel blocks, pitch 16
    (2, 20, 24, 192, 64, 3, 3, (1, 1), (1, 1)),    # three channel blocks
    (1, 16, 32, 128, 128, 2, 3, (1, 1), (1, 1)),   # R != S
]


@pytest.mark.parametrize("case", STREAM_CASES, ids=lambda c: "x".join(map(str, c[:7])))
@pytest.mark.parametrize("out_dt", ["f32", "bf16"])
def test_window_stream_exact(alcop, case, out_dt):
    X, Wt, ref = _inputs(case, 101)
    _, _, _, C, K, R, S, st, pd = case
    odt = torch.float32 if out_dt == "f32" else torch.bfloat16
    want = torch.from_numpy(ref).to(odt)
    d = alcop.conv_desc(*case[:7], st, pd, alcop.BF16, alcop.F32 if out_dt == "f32" else alcop.BF16)
    pick = alcop.choose_conv_schedule(d)
    assert pick.tileN == K, pick
    scheds = [pick]
    for tk in (64, 64 * S):
        for sa, sb in ((1, 2), (2, 3), (2, 1)):
            scheds.append(alcop.make_schedule(tileN=K, tileK=tk, n_stage=sa, n_stage_B=sb, n_stage_inner=2))
    # schedules only the streamed-filter kernel accepts (a chunk of S taps, or unequal A / B rings: the
    # im2col kernel needs tileK 64 and equal stages), so a pass proves that kernel ran
    only_streamed = [alcop.make_schedule(tileN=K, tileK=64 * S, n_stage=2, n_stage_B=1, n_stage_inner=2),
                     alcop.make_schedule(tileN=K, tileK=64, n_stage=1, n_stage_B=2, n_stage_inner=1)]
    for s in only_streamed:
        Y = alcop.conv2d(X, Wt, st, pd, sched=s, out_dtype=odt)
        _assert_equal(Y.cpu(), want, "streamed %s" % s)
    for s in scheds:
        try:
            Y = alcop.conv2d(X, Wt, st, pd, sched=s, out_dtype=odt)
        except alcop.AlcopError as e:
            assert "SmemCapacity" in str(e) or "BadSchedule" in str(e), (s, e)  # a ring too deep for this K
            continue
        _assert_equal(Y.cpu(), want, "streamed %s" % s)


# ----------------------------------------------------------------------------
# Window modes on CTA pairs (cta_group 2): a 256-pixel tile = the two CTAs'
# TR-row windows, one tcgen05.mma.cta_group::2 (M = 256) per k-step issued by
# the leader, each CTA staging half of the filter rows (resident or streamed).
# Odd tile-row counts leave the last pair's peer rows outside the image.
@pytest.mark.parametrize("case", WINDOW_CASES, ids=lambda c: "x".join(map(str, c[:7])) + "_p%d%d" % c[8])
def test_window_pairs_exact(alcop, case):
    X, Wt, ref = _inputs(case, 95)
    _, _, _, _, K, _, _, st, pd = case
    ran = 0
    for out_dt in ("f32", "bf16"):
        odt = torch.float32 if out_dt == "f32" else torch.bfloat16
        want = torch.from_numpy(ref).to(odt)
        for stages, inner in ((2, 2), (3, 1), (4, 4), (1, 2)):
            s = alcop.make_schedule(tileN=K, tileK=64, n_stage=stages, n_stage_inner=inner, mode=1, cta_group=2)
            try:
                Y = alcop.conv2d(X, Wt, st, pd, sched=s, out_dtype=odt)
            except alcop.AlcopError as e:
                assert "SmemCapacity" in str(e) or "TmemCapacity" in str(e), (s, e)
                continue
            ran += 1
            _assert_equal(Y.cpu(), want, "window pair %s" % s)
    assert ran >= 4


def test_window_pairs_small_grid(alcop):
    """Two clusters walking every pair tile of three images (the cursor's
    carries across images), resident filter and streamed filter."""
    for case, sched in (((3, 28, 28, 64, 64, 3, 3, (1, 1), (1, 1)),
                         dict(tileN=64, tileK=64, n_stage=2, n_stage_inner=2)),
                        ((3, 28, 28, 128, 128, 3, 3, (1, 1), (1, 1)),
                         dict(tileN=128, tileK=64, n_stage=2, n_stage_B=3, n_stage_inner=2))):
        X, Wt, ref = _inputs(case, 97)
        s = alcop.make_schedule(cta_group=2, **sched)
        s.num_ctas = 4
        Y = alcop.conv2d(X, Wt, (1, 1), (1, 1), sched=s, out_dtype=torch.float32)
        _assert_equal(Y.cpu(), torch.from_numpy(ref), "pair grid 4 %s" % (case[:7],))


@pytest.mark.parametrize("case", STREAM_CASES, ids=lambda c: "x".join(map(str, c[:7])))
def test_window_stream_pairs_exact(alcop, case):
    X, Wt, ref = _inputs(case, 103)
    _, _, _, C, K, R, S, st, pd = case
    want = torch.from_numpy(ref).to(torch.bfloat16)
    # unequal A / B rings or an S-tap filter chunk: only the streamed-filter kernel accepts them
    for tk, sa, sb in ((64, 1, 2), (64 * S, 2, 1), (64, 2, 4), (64 * S, 1, 2)):
        s = alcop.make_schedule(tileN=K, tileK=tk, n_stage=sa, n_stage_B=sb, n_stage_inner=2, cta_group=2)
        try:
            Y = alcop.conv2d(X, Wt, st, pd, sched=s, out_dtype=torch.bfloat16)
        except alcop.AlcopError as e:
            assert "SmemCapacity" in str(e), (s, e)
            continue
        _assert_equal(Y.cpu(), want, "streamed pair %s" % s)
