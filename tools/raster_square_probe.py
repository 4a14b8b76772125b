"""C5 squares on the 256x512 CTA-pair tile under several raster groups
(schedule.raster = tile rows per group; 0 = the auto group): sustained time
(each measurement ~1 s of back-to-back launches, round-robin over the groups,
median of 3) — measurement tool for the HBM re-read factor of the big squares.

python tools/raster_square_probe.py [n ...]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2210_16691_b200 as alcop
from paper_2210_16691_b200.timing import time_graph

ns = [int(v) for v in sys.argv[1:]] or [16384, 12288]
out = {}
for n in ns:
    A = (torch.rand(n, n, device="cuda") - 0.5).to(torch.bfloat16)
    B = (torch.rand(n, n, device="cuda") - 0.5).to(torch.bfloat16)
    C = torch.empty(n, n, device="cuda", dtype=torch.bfloat16)
    base = alcop.choose_schedule(alcop.gemm_desc(n, n, n))
    groups = (0, 2, 4, 6, 8, 16, 32, 64)
    res = {g: [] for g in groups}
    fl = 2.0 * n ** 3
    for rnd in range(3):
        for g in groups:
            s = alcop.make_schedule(tileN=base.tileN, tileK=base.tileK, n_stage=base.n_stage_smem_A,
                                    n_stage_inner=base.n_stage_inner, cta_group=base.cta_group, raster=g)
            per = max(1, int(1.0 / (fl / 1.4e15)))  # ~1 s of launches
            res[g].append(time_graph(lambda i: alcop.matmul(A, B, s, out=C), iters=per, warmup=2))
    out[str(n)] = {"schedule": str(base),
                   **{("auto" if g == 0 else "G%d" % g): round(fl / sorted(v)[1] / 1e9, 1) for g, v in res.items()}}
    print(json.dumps({n: out[str(n)]}), flush=True)
    del A, B, C
    torch.cuda.empty_cache()
