"""Fits the power-capped terms of the B200 model (alcop_hw.tCapFlop,
tCapL2Byte, tCapDramByte) to the sustained-regime measurements in
profiles/power_r02.json (tools/power_probe.py): time = tCapFlop * FLOPs +
tCapL2Byte * L2->SM bytes + tCapDramByte * DRAM bytes, with the bytes as the
model itself estimates them (alcop_predict's bytesL2 / bytesDram), by
non-negative least squares on relative error.  Prints the constants and the
per-point error; --check compares the compiled defaults against the fit.

    python tools/fit_power.py [--check]"""
import json
import os
import sys

import numpy as np
from scipy.optimize import nnls

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2210_16691_b200 as alcop  # noqa: E402


def rows():
    d = json.load(open(os.path.join(ROOT, "profiles", "power_r02.json")))
    hw = alcop.hw_b200()
    hw.tCapFlop = hw.tCapL2Byte = hw.tCapDramByte = 0.0
    out = []
    for p in d["points"]:
        n = p["n"]
        desc = alcop.gemm_desc(n, n, n, 1, alcop.BF16, alcop.BF16, alcop.B_KN)
        s = alcop.default_schedule(**p["schedule"])
        b = alcop.predict(desc, s, hw)
        out.append((p, b))
    return out


def design(data):
    X = np.array([[2.0 * p["n"] ** 3, b["bytesL2"], b["bytesDram"]] for p, b in data])
    y = np.array([p["ms_sustained"] * 1e-3 for p, b in data])
    return X, y


def fit(X, y):
    w = 1.0 / y  # relative error
    coef, _ = nnls(X * w[:, None], y * w)
    return coef


def held_out(data):
    """Leave one problem size out: fit on the others, relative errors on it."""
    out = {}
    sizes = sorted(set(p["n"] for p, _ in data))
    for n in sizes:
        tr = [d for d in data if d[0]["n"] != n]
        te = [d for d in data if d[0]["n"] == n]
        c = fit(*design(tr))
        X, y = design(te)
        out[n] = list((X @ c - y) / y)
    return out


def main():
    data = rows()
    X, y = design(data)
    coef = fit(X, y)
    pred = X @ coef
    err = (pred - y) / y
    print("tCapFlop %.4e s/FLOP  tCapL2Byte %.4e s/B  tCapDramByte %.4e s/B" % tuple(coef))
    print("rms rel err %.3f  max %.3f" % (np.sqrt(np.mean(err ** 2)), np.max(np.abs(err))))
    for (p, b), e in zip(data, err):
        print("%6d %-14s meas %.3f ms  fit %+.1f%%  dram est %.1f GB meas %.1f GB  l2 %.1f GB" % (
            p["n"], p["sched"], p["ms_sustained"], 100 * e, b["bytesDram"] / 1e9, p["dram_B"] / 1e9,
            b["bytesL2"] / 1e9))
    for n, e in held_out(data).items():
        print("held out n=%d: rms %.3f max %.3f" % (n, np.sqrt(np.mean(np.square(e))), np.max(np.abs(e))))
    if "--check" in sys.argv:
        hw = alcop.hw_b200()
        got = np.array([hw.tCapFlop, hw.tCapL2Byte, hw.tCapDramByte])
        assert np.allclose(got, coef, rtol=0.02), (got, coef)
        print("compiled defaults match the fit")


if __name__ == "__main__":
    main()
