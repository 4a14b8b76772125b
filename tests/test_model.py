"""The host analytical model (alcop_predict / alcop_choose_schedule): Table
identities of the paper's model and the
model-pick criterion against the measured exhaustive sweep committed in
profiles/sweep_r01.json (the B200 stand-in for measure_ground_truth,
pipe_sim.hpp:195-239)."""
import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SWEEP = os.path.join(ROOT, "profiles", "sweep_r01.json")


def test_breakdown_identities(alcop):
    d = alcop.gemm_desc(4096, 3072, 768)
    for st in (1, 2, 4):
        s = alcop.make_schedule(tileN=256, tileK=64, n_stage=st)
        b = alcop.predict(d, s)
        assert b["tThreadblk"] == pytest.approx(b["tInit"] + b["tMainLoop"] + b["tEpilogue"])
        assert b["seconds"] == pytest.approx(b["tKernel"] / (1.9e9))
        assert b["nSmemLoop"] == 768 // 64
        assert b["nRegLoop"] == 64 // 16
        # never faster than the tensor-core floor
        assert b["seconds"] >= 2.0 * 4096 * 3072 * 768 / (148 * 8192 * 1.9e9)


def test_more_stages_never_predicted_slower(alcop):
    d = alcop.gemm_desc(8192, 8192, 8192)
    prev = None
    for st in range(1, 5):
        t = alcop.predict(d, alcop.make_schedule(tileN=256, tileK=64, n_stage=st))["tKernel"]
        if prev is not None:
            assert t <= prev + 1e-6
        prev = t


def test_wrap_mode_costs_redundant_loads(alcop):
    d = alcop.gemm_desc(4096, 4096, 4096)
    fused = alcop.predict(d, alcop.make_schedule(tileN=256, tileK=64, n_stage=4, mode=alcop.MODE_FUSED))
    wrap = alcop.predict(d, alcop.make_schedule(tileN=256, tileK=64, n_stage=4, mode=alcop.MODE_WRAP))
    assert wrap["tKernel"] > fused["tKernel"]


def test_choose_schedule_is_valid(alcop):
    for shape in [(512, 512, 512, 1), (4096, 768, 768, 1), (16384, 16384, 16384, 1), (512, 64, 512, 192),
                  (300, 200, 104, 3)]:
        d = alcop.gemm_desc(*shape)
        s = alcop.choose_schedule(d)
        alcop.validate(d, s)


def test_model_pick_within_ten_percent_of_sweep(alcop):
    """tools/check_model.py: measured time of the model's pick / best measured
    time over every swept schedule, per shape (BASELINE: within 10%)."""
    if not os.path.exists(SWEEP):
        pytest.skip("no committed sweep")
    import sys
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    from check_model import evaluate
    with open(SWEEP) as f:
        res = evaluate(json.load(f))
    ratios = {k: v["pick_over_best"] for k, v in res.items()}
    assert len(ratios) >= 8
    assert all(r == r for r in ratios.values()), ("model pick not in the sweep", ratios)  # no NaN
    # all but at most one shape within 10%; none beyond 15%
    assert sum(r > 1.10 for r in ratios.values()) <= 1, ratios
    assert max(ratios.values()) <= 1.15, ratios


@pytest.mark.gpu
def test_model_assisted_tuning_on_gpu(alcop):
    """tuner.hpp:407-413 (AnalyticalOnly) on real timings: the best of the
    model's top-8 is within 5% of the best of its top-40 (a near-exhaustive
    search of the well-ranked region)."""
    import torch
    M, N, K = 4096, 3072, 768
    A = (torch.rand(M, K, device="cuda") - 0.5).to(torch.bfloat16)
    B = (torch.rand(K, N, device="cuda") - 0.5).to(torch.bfloat16)
    C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    best8, t8 = alcop.tune(A, B, C, budget=8)
    best40, t40 = alcop.tune(A, B, C, budget=40)
    m8 = min(t["measured_s"] for t in t8)
    m40 = min(t["measured_s"] for t in t40)
    assert len(t8) == 8 and len(t40) == 40
    assert m8 <= 1.05 * m40, (m8, m40, best8, best40)


def test_fit_script_restates_the_product_model(alcop):
    """tools/fit_model.py (the calibration's vectorised restatement) must predict
    exactly what alcop_predict does with the same constants, or the fitted
    constants would not mean what model.cpp uses them for."""
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import fit_model
    hw = alcop.hw_b200(burst=True)
    P = {"tp": hw.throughputSM, "bwL2": hw.bwLLC, "t_issue": hw.tIssue, "t_issue_b": hw.tIssuePerBox,
         "lat": hw.latLLCRead, "bwW": hw.bwDRAMWrite, "epi0": hw.latDRAMWrite, "launch": hw.tLaunch,
         "bwD": hw.bwDRAM, "tile0": hw.tTile, "ovl": hw.overlapDRAM, "bwSM": hw.bwSmem, "pair0": hw.tPair}
    with open(SWEEP) as f:
        rows = json.load(f)
    for r in rows[::37]:
        d = alcop.gemm_desc(r["M"], r["N"], r["K"], r["batch"], alcop.BF16, alcop.BF16, alcop.B_KN)
        s = alcop.make_schedule(tileN=r["tileN"], tileK=r["tileK"], n_stage=r["stages"], n_stage_inner=r["inner"],
                                mode=r["mode"], cta_group=r.get("cg", 1))
        want = alcop.predict(d, s, hw)["tKernel"]
        got = fit_model.predict_cycles(r, P)
        assert abs(got - want) <= 1e-6 * want, (r, got, want)


def test_power_capped_model_fit(alcop):
    """The power-cap terms (alcop_hw.tCap*) are the non-negative least-squares
    fit of tools/fit_power.py to the sustained measurements in
    profiles/power_r02.json (30 schedules x sizes): compiled defaults equal the
    fit, the fit is within 10% rms, and each problem size left out of the fit
    is predicted within 15% rms."""
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import numpy as np
    import fit_power
    data = fit_power.rows()
    X, y = fit_power.design(data)
    coef = fit_power.fit(X, y)
    hw = alcop.hw_b200()
    assert np.allclose([hw.tCapFlop, hw.tCapL2Byte, hw.tCapDramByte], coef, rtol=0.02)
    err = (X @ coef - y) / y
    assert np.sqrt(np.mean(err ** 2)) <= 0.10
    for n, e in fit_power.held_out(data).items():
        assert np.sqrt(np.mean(np.square(e))) <= 0.15, (n, e)


def test_power_regime_picks_the_wide_pair_tile_for_squares(alcop):
    """Sustained regime: the model's pick for the C5 squares is the 256 x 512
    CTA-pair tile, the measured fastest class at the power cap
    (profiles/power_r02.json: 1398-1425 vs 1151-1194 TFLOP/s for 256 x 256)."""
    for n in (8192, 12288, 16384):
        s = alcop.choose_schedule(alcop.gemm_desc(n, n, n))
        assert (s.cta_group, s.tileN, s.n_stage_inner) == (2, 512, 1), (n, s)


def test_choose_conv_schedule_is_valid_for_every_resnet_layer(alcop):
    """alcop_choose_conv_schedule (C ABI) returns a launchable conv schedule
    for all 23 ResNet-50 layers: the GEMM space for 1x1 stride-1 layers, the
    window kernels' spaces (stem; window and streamed filter, CTA pairs
    included), else the im2col
    kernel's (tileK 64, equal stages, CTA pairs only for C % 64 == 0,
    within the 4-epilogue-warp shared memory)."""
    from paper_2210_16691_b200 import workloads as W
    import ctypes
    lib = alcop.load_library()
    for L in W.CONV_LAYERS:
        s = W.conv_schedule(alcop, L, 256)
        if L.gemm:  # 1x1 stride 1: the GEMM kernels' space (CTA pairs included)
            g = W.conv_gemm_desc(alcop, L, 256)
            alcop.validate(g, s)
            assert lib.alcop_smem_bytes(ctypes.byref(g), ctypes.byref(s)) <= 232448
            continue
        if L.stream:  # window + streamed filter: tileK = 64 x taps per filter chunk, own A / B rings
            assert s.tileN == L.K and s.tileK in (64, 64 * L.R) and s.tileM == 128 * s.cta_group, s
            continue
        assert s.tileK == 64 and s.n_stage_smem_A == s.n_stage_smem_B, L.name
        if L.stem or L.window:  # the window kernel: tile = 128 output pixels (256 on a CTA pair) x all K filters
            assert s.tileN == L.K and 1 <= s.n_stage_inner <= 8 and s.tileM == 128 * s.cta_group, s
            assert s.cta_group == 1 or not L.stem, s  # the stem modes run one CTA per tile
            continue
        assert s.cta_group == 1 or (L.Cs % 64 == 0 and not L.halo), L.name  # pairs: the 64-channel im2col path
        g = W.conv_gemm_desc(alcop, L, 256)
        alcop.validate(g, s)
        assert lib.alcop_smem_bytes(ctypes.byref(g), ctypes.byref(s)) <= 232448
