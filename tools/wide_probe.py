"""Burst per-GEMM times of the model pick, the 256x512 CTA-pair tile (tileN 512,
raster groups) and cuBLAS on the squares, 5 round-robin rounds, median
(measurement tool)."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2210_16691_b200 as alcop  # noqa: E402
from paper_2210_16691_b200 import workloads as W  # noqa: E402
from paper_2210_16691_b200.timing import time_graph  # noqa: E402

out = {}
for n in W.SQUARES:
    A = (torch.rand(n, n, device="cuda") - 0.5).to(torch.bfloat16)
    B = (torch.rand(n, n, device="cuda") - 0.5).to(torch.bfloat16)
    C = torch.empty(n, n, device="cuda", dtype=torch.bfloat16)
    cands = {"pick": W.square_schedule(alcop, n, n)}
    for st in (3, 4):
        for r in (0, 4, 8, 16):
            cands["wide_s%d_r%d" % (st, r)] = alcop.make_schedule(tileN=512, tileK=64, n_stage=st, n_stage_inner=1,
                                                                  cta_group=2, raster=r)
    cands["wide_bk128_s2"] = alcop.make_schedule(tileN=512, tileK=128, n_stage=2, n_stage_inner=1, cta_group=2)
    fns = {k: (lambda i, s=s: alcop.matmul(A, B, s, out=C)) for k, s in cands.items()}
    fns["cublas"] = lambda i: torch.matmul(A, B, out=C)
    it = 20 if n <= 4096 else (6 if n <= 8192 else 3)
    t = {k: [] for k in fns}
    for _ in range(5):
        for k, f in fns.items():
            t[k].append(time_graph(f, iters=it, warmup=1))
    out[str(n)] = {k: round(2.0 * n ** 3 / statistics.median(v) / 1e9, 1) for k, v in t.items()}
    print(json.dumps({str(n): out[str(n)]}), flush=True)
