"""Fits the B200 analytical model's hardware constants to a measured sweep
(profiles/sweep_r01.json) and reports the model-pick quality per shape.

The model form is the one model.cpp implements (B200 view of PAPER.md
Table "Analytical Performance Model"); this script only chooses its
constants.  python tools/fit_model.py profiles/sweep_r01.json
"""
import json
import math
import sys
from collections import defaultdict

import numpy as np
from scipy.optimize import minimize

NSM = 148


def pipeline_latency(tLoad, tUse, n, nPipe):
    # perf_model.hpp:53-57 with nMplx = 1 (one CTA per SM); numpy-vectorised
    return np.where(tLoad <= (nPipe - 1) * tUse, tUse * n, (tLoad + tUse) * n / nPipe)


def features(rows):
    """Per-row arrays of everything the model needs that does not depend on
    the constants (B[K,N] layout, as the sweep measures)."""
    f = defaultdict(list)
    for r in rows:
        M, N, K, b = r["M"], r["N"], r["K"], r["batch"]
        BN, BK, s, inner, mode = r["tileN"], r["tileK"], r["stages"], r["inner"], r["mode"]
        cg = r.get("cg", 1)
        tiles = math.ceil(M / (128 * cg)) * math.ceil(N / BN) * b
        units = min(tiles, NSM // cg)   # CTAs (pairs) working at once
        bN = BN // cg                     # B columns per CTA
        # pair halves of 96 columns: two 64-column atoms when that fits (alcop_api.cpp pair_b_pad)
        pad = cg == 2 and bN % 64 != 0 and (1024 + s * (128 * BK * 2 + 128 * BK * 2)
                                            + 8 * (5 * s + 4) + 16 + 4 * 32 * 128) <= 232448
        bcols = 128 if pad else bN
        a_boxes = 1 if (BK > 64 and K % 64 == 0) else max(1, BK // 64)   # atom-stacked view
        b_boxes = 2 if pad else (bN // 32 if bN % 64 else max(1, bN // 64))
        for k, v in (("ctas", units * cg), ("waves", math.ceil(tiles / units)), ("E", math.ceil(K / BK)),
                     ("bytes_kb", (128 + bcols) * BK * 2), ("mma", 2 * 128 * BN * BK), ("boxes", a_boxes + b_boxes),
                     ("s", s), ("inner", inner), ("mode", mode), ("cg", cg), ("BN", BN),
                     ("dram_bytes", (M * K + K * N + M * N) * 2 * b), ("ms", r["ms"])):
            f[k].append(v)
    return {k: np.array(v, dtype=np.float64) for k, v in f.items()}


def predict_cycles_v(F, P):
    """model.cpp alcop_predict, vectorised over the sweep rows."""
    t_mma = F["mma"] / P["tp"]
    t_l2 = np.maximum(F["bytes_kb"] * F["ctas"] / P["bwL2"], F["bytes_kb"] / P["bwSM"])
    t_kb = np.maximum(np.maximum(t_mma, t_l2), P["t_issue"] + P["t_issue_b"] * F["boxes"])
    loads = F["E"] + np.where(F["mode"] == 0, F["s"] - 1, 0)
    main = pipeline_latency(P["lat"], t_kb, loads, F["s"]) + P["tile0"]
    main = main + np.where((F["mode"] == 0) | (F["s"] == 1), P["lat"] * 0.5, 0.0)  # per-tile refill bubble
    epi = 128 * F["BN"] * 2 * F["ctas"] / P["bwW"] + P["epi0"]
    body = np.where(F["inner"] >= 2, F["waves"] * np.maximum(main, epi) + np.minimum(main, epi),
                    F["waves"] * (main + epi))
    t = P["lat"] + body + np.where(F["cg"] == 2, P["pair0"], 0.0)
    dram = F["dram_bytes"] / P["bwD"]
    # DRAM and the SM pipeline overlap imperfectly: soft maximum
    return P["launch"] + np.maximum(t, dram) + P["ovl"] * np.minimum(t, dram)


def predict_cycles(r, P):
    return float(predict_cycles_v(features([r]), P)[0])


KEYS = ["tp", "bwL2", "t_issue", "t_issue_b", "lat", "bwW", "epi0", "launch", "bwD", "tile0", "ovl", "bwSM", "pair0"]
INIT = {"tp": 8192.0, "bwL2": 6500.0, "t_issue": 250.0, "t_issue_b": 20.0, "lat": 1800.0, "bwW": 3000.0,
        "epi0": 800.0, "launch": 3000.0, "bwD": 3300.0, "tile0": 300.0, "ovl": 0.2, "bwSM": 80.0, "pair0": 500.0}
CLOCK = 1.9e9
PICK_W = 0.0


def load(path):
    with open(path) as f:
        return json.load(f)


FIXED = {}


def loss(x, F, groups):
    """rms log error + a pick-quality term (mean log(pick/best) over shapes)."""
    P = dict(zip([k for k in KEYS if k not in FIXED], np.exp(x)))
    P.update(FIXED)
    pc = predict_cycles_v(F, P)
    err = np.log(pc / CLOCK * 1e3) - np.log(F["ms"])
    pick = 0.0
    for idx in groups:
        pick += math.log(F["ms"][idx][np.argmin(pc[idx])] / F["ms"][idx].min())
    return math.sqrt(float(np.mean(err ** 2))) + PICK_W * pick / len(groups)


def report(rows, P):
    by = defaultdict(list)
    for r in rows:
        by[(r["M"], r["N"], r["K"], r["batch"])].append(r)
    worst = 1.0
    for k, v in by.items():
        best = min(v, key=lambda r: r["ms"])
        pick = min(v, key=lambda r: predict_cycles(r, P))
        ratio = pick["ms"] / best["ms"]
        worst = max(worst, ratio)
        pred_best = predict_cycles(best, P) / CLOCK * 1e3
        print("%-22s best %.4f ms (%d,%d,s%d,t%d,m%d,cg%d) pick %.4f ms (%d,%d,s%d,t%d,m%d,cg%d) ratio %.3f  pred(best) %.4f"
              % (k, best["ms"], best["tileN"], best["tileK"], best["stages"], best["inner"], best["mode"],
                 best.get("cg", 1), pick["ms"], pick["tileN"], pick["tileK"], pick["stages"], pick["inner"],
                 pick["mode"], pick.get("cg", 1), ratio, pred_best))
    print("worst pick/best:", round(worst, 3))


def main():
    global PICK_W
    rows = load(sys.argv[1])
    for a in sys.argv[2:]:
        k, v = a.split("=")
        if k == "pick_w":
            PICK_W = float(v)
        else:
            FIXED[k] = float(v)
    free = [k for k in KEYS if k not in FIXED]
    x0 = np.log([INIT[k] for k in free])
    F = features(rows)
    by = defaultdict(list)
    for i, r in enumerate(rows):
        by[(r["M"], r["N"], r["K"], r["batch"])].append(i)
    groups = [np.array(v) for v in by.values()]
    best = None
    for trial in range(8):
        start = x0 + (np.random.RandomState(trial).randn(len(x0)) * 0.3 if trial else 0)
        res = minimize(loss, start, args=(F, groups), method="Nelder-Mead",
                       options={"maxiter": 8000, "xatol": 1e-4, "fatol": 1e-7})
        if best is None or res.fun < best.fun:
            best = res
    res = best
    P = dict(zip(free, np.exp(res.x)))
    P.update(FIXED)
    print("fit objective:", res.fun)
    print(json.dumps({k: round(v, 2) for k, v in P.items()}))
    report(rows, P)


if __name__ == "__main__":
    main()
