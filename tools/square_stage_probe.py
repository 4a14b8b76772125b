"""C5 squares: ring depth of the 256x512 CTA-pair tile (and the 256x256 tile)
timed two ways — burst (a short CUDA graph, the GPU cool) and sustained (~1 s
of back-to-back launches, power-capped) — round-robin over the schedules,
median of 3.  Measurement tool: python tools/square_stage_probe.py [n ...]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2210_16691_b200 as alcop
from paper_2210_16691_b200.timing import time_graph

ns = [int(v) for v in sys.argv[1:]] or [16384, 8192]
for n in ns:
    A = (torch.rand(n, n, device="cuda") - 0.5).to(torch.bfloat16)
    B = (torch.rand(n, n, device="cuda") - 0.5).to(torch.bfloat16)
    C = torch.empty(n, n, device="cuda", dtype=torch.bfloat16)
    fl = 2.0 * n ** 3
    cands = {"w_s%d" % st: alcop.make_schedule(tileN=512, tileK=32, n_stage=st, n_stage_inner=1, cta_group=2)
             for st in (3, 4, 5, 6, 8)}
    cands.update({"p256_s%d" % st: alcop.make_schedule(tileN=256, tileK=64, n_stage=st, cta_group=2) for st in (4, 6)})
    res = {k: {"burst": [], "sustained": []} for k in cands}
    burst_iters = max(2, int(0.02 / (fl / 1.6e15)))
    sus_iters = max(4, int(1.0 / (fl / 1.4e15)))
    for rnd in range(3):
        for k, s in cands.items():
            res[k]["burst"].append(time_graph(lambda i: alcop.matmul(A, B, s, out=C), iters=burst_iters, warmup=1))
            torch.cuda.synchronize()
            torch.cuda._sleep(int(2e9))  # ~1 s idle: cool down before the next burst sample
        for k, s in cands.items():
            res[k]["sustained"].append(time_graph(lambda i: alcop.matmul(A, B, s, out=C), iters=sus_iters, warmup=2))
    out = {k: {m: round(fl / sorted(v)[1] / 1e9, 1) for m, v in r.items()} for k, r in res.items()}
    out["model_pick"] = str(alcop.choose_schedule(alcop.gemm_desc(n, n, n)))
    print(json.dumps({n: out}), flush=True)
    del A, B, C
    torch.cuda.empty_cache()
