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
    # perf_model.hpp:53-57 with nMplx = 1 (one CTA per SM)
    if tLoad <= (nPipe - 1) * tUse:
        return tUse * n
    return (tLoad + tUse) * n / nPipe


def predict_cycles(r, P):
    """P = dict of constants (cycles / bytes-per-cycle)."""
    M, N, K, b = r["M"], r["N"], r["K"], r["batch"]
    BN, BK, s, inner, mode = r["tileN"], r["tileK"], r["stages"], r["inner"], r["mode"]
    cg = r.get("cg", 1)
    tiles = math.ceil(M / (128 * cg)) * math.ceil(N / BN) * b
    units = min(tiles, NSM // cg)   # CTAs (pairs) working at once
    ctas = units * cg
    waves = math.ceil(tiles / units)
    E = math.ceil(K / BK)
    bytes_kb = (128 + BN // cg) * BK * 2   # per CTA
    t_mma = 2 * 128 * BN * BK / P["tp"]
    t_l2 = max(bytes_kb * ctas / P["bwL2"], bytes_kb / P["bwSM"])
    boxes = max(1, BK // 64) + max(1, (BN // cg) // 64)
    t_kb = max(t_mma, t_l2, P["t_issue"] + P["t_issue_b"] * boxes)
    loads = E + (s - 1 if mode == 0 else 0)
    main = pipeline_latency(P["lat"], t_kb, loads, s) + P["tile0"]
    if mode == 0 or s == 1:
        main += P["lat"] * 0.5  # per-tile refill bubble
    epi = 128 * BN * 2 * ctas / P["bwW"] + P["epi0"]
    if inner >= 2:
        body = waves * max(main, epi) + min(main, epi)
    else:
        body = waves * (main + epi)
    t = P["lat"] + body + (P["pair0"] if cg == 2 else 0.0)
    dram = (M * K + K * N + M * N) * 2 * b / P["bwD"]
    # DRAM and the SM pipeline overlap imperfectly: soft maximum
    return P["launch"] + max(t, dram) + P["ovl"] * min(t, dram)


KEYS = ["tp", "bwL2", "t_issue", "t_issue_b", "lat", "bwW", "epi0", "launch", "bwD", "tile0", "ovl", "bwSM", "pair0"]
INIT = {"tp": 8192.0, "bwL2": 6500.0, "t_issue": 250.0, "t_issue_b": 20.0, "lat": 1800.0, "bwW": 3000.0,
        "epi0": 800.0, "launch": 3000.0, "bwD": 3300.0, "tile0": 300.0, "ovl": 0.2, "bwSM": 80.0, "pair0": 500.0}
CLOCK = 1.9e9
PICK_W = 0.0


def load(path):
    with open(path) as f:
        return json.load(f)


FIXED = {}


def loss(x, rows):
    """rms log error + a pick-quality term (mean log(pick/best) over shapes)."""
    P = dict(zip(KEYS, np.exp(x)))
    P.update(FIXED)
    err = 0.0
    by = defaultdict(list)
    for r in rows:
        pc = predict_cycles(r, P)
        err += (math.log(pc / CLOCK * 1e3) - math.log(r["ms"])) ** 2
        by[(r["M"], r["N"], r["K"], r["batch"])].append((pc, r["ms"]))
    pick = 0.0
    for v in by.values():
        best = min(m for _, m in v)
        chosen = min(v)[1]
        pick += math.log(chosen / best)
    return math.sqrt(err / len(rows)) + PICK_W * pick / len(by)


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
    x0 = np.log([INIT[k] for k in KEYS])
    best = None
    for trial in range(6):
        start = x0 + (np.random.RandomState(trial).randn(len(x0)) * 0.3 if trial else 0)
        res = minimize(loss, start, args=(rows,), method="Nelder-Mead",
                       options={"maxiter": 4000, "xatol": 1e-4, "fatol": 1e-7})
        if best is None or res.fun < best.fun:
            best = res
    res = best
    P = dict(zip(KEYS, np.exp(res.x)))
    P.update(FIXED)
    print("fit objective:", res.fun)
    print(json.dumps({k: round(v, 2) for k, v in P.items()}))
    report(rows, P)


if __name__ == "__main__":
    main()
