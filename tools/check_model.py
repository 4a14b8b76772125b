"""Model-pick quality of the product model (libalcop alcop_predict /
alcop_choose_schedule) against a measured sweep: for every shape, the
measured time of the model's pick over the best measured time (the paper's
'model pick within 10% of exhaustive tuning' criterion)."""
import json, os, sys
from collections import defaultdict
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2210_16691_b200 as alcop


def evaluate(rows, hw=None):
    """rows: a burst-regime sweep (profiles/sweep_r01.json: each schedule timed
    in short graphs); the model is evaluated in the same regime (power-cap
    terms off, alcop.hw_b200(burst=True)) unless `hw` is given."""
    hw = hw or alcop.hw_b200(burst=True)
    by = defaultdict(list)
    for r in rows:
        by[(r["M"], r["N"], r["K"], r["batch"])].append(r)
    out = {}
    for (M, N, K, b), v in by.items():
        d = alcop.gemm_desc(M, N, K, b, alcop.BF16, alcop.BF16, alcop.B_KN)
        best = min(v, key=lambda r: r["ms"])
        pick = alcop.choose_schedule(d, hw)
        meas = [r for r in v if (r["tileN"], r["tileK"], r["stages"], r["inner"], r["mode"], r.get("cg", 1)) ==
                (pick.tileN, pick.tileK, pick.n_stage_smem_A, pick.n_stage_inner, pick.mode, pick.cta_group)]
        pm = meas[0]["ms"] if meas else float("nan")
        pred = alcop.predict(d, pick, hw)["seconds"] * 1e3
        out["%dx%dx%dx%d" % (M, N, K, b)] = {"best_ms": best["ms"], "best": [best["tileN"], best["tileK"], best["stages"], best["inner"], best["mode"], best.get("cg", 1)],
                                              "pick_ms": pm, "pick": [pick.tileN, pick.tileK, pick.n_stage_smem_A, pick.n_stage_inner, pick.mode, pick.cta_group],
                                              "pred_ms": pred, "pick_over_best": pm / best["ms"]}
    return out


if __name__ == "__main__":
    res = evaluate(json.load(open(sys.argv[1])))
    for k, v in res.items():
        print("%-20s best %.4f %s  pick %.4f %s  ratio %.3f  pred %.4f" % (k, v["best_ms"], v["best"], v["pick_ms"], v["pick"], v["pick_over_best"], v["pred_ms"]))
    print("worst:", max(v["pick_over_best"] for v in res.values()))
