"""alcop_tune on one GEMM view (measurement tool): the first-pass ranking of
its top candidates, the pick, and the pick re-timed against given schedules.
python tools/tune_probe.py M N K [budget] [tn,tk,st,cg ...]   (B as [N, K], K-major)"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2210_16691_b200 as alcop
from paper_2210_16691_b200.timing import time_graph

M, N, K = map(int, sys.argv[1:4])
budget = int(sys.argv[4]) if len(sys.argv) > 4 else 24
X = (torch.rand(M, K, device="cuda") - 0.5).to(torch.bfloat16)
W = (torch.rand(N, K, device="cuda") - 0.5).to(torch.bfloat16)
Y = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
best, trials = alcop.tune(X, W, Y, budget=budget, b_layout=alcop.B_NK)
fl = 2.0 * M * N * K
first = sorted(trials, key=lambda t: t["measured_s"])[:8]
out = {"pick": str(best), "top8 (first pass; the shortlist re-timed)": [
    (t["schedule"]["tileN"], t["schedule"]["tileK"], t["schedule"]["n_stage_smem_A"], t["schedule"]["cta_group"],
     round(fl / t["measured_s"] / 1e12, 1)) for t in first]}
others = {}
for spec in sys.argv[5:]:
    tn, tk, st, cg = map(int, spec.split(","))
    others[spec] = alcop.make_schedule(tileN=tn, tileK=tk, n_stage=st, cta_group=cg, n_stage_inner=1 if tn == 512 else 2)
others["pick"] = best
res = {k: [] for k in others}
for _ in range(3):
    for k, s in others.items():
        res[k].append(time_graph(lambda i, s=s: alcop.matmul(X, W, s, b_layout=alcop.B_NK, out=Y), iters=40,
                                 warmup=2))
out["retimed"] = {k: round(fl / sorted(v)[1] / 1e9, 1) for k, v in res.items()}
print(json.dumps(out))
