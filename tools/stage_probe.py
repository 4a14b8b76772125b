"""Stage-depth probe: one tile shape, tileK 32/64/128 x every stage count that
fits, CUDA-graph timing on rotating cold inputs (measurement tool).
Usage: python tools/stage_probe.py M N K tileN cta_group"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2210_16691_b200 as alcop
from paper_2210_16691_b200.timing import Rotating, time_graph

M, N, K, tn, cg = map(int, sys.argv[1:6])
rot = Rotating(lambda i: ((torch.rand(M, K, device="cuda") - 0.5).to(torch.bfloat16),
                          (torch.rand(K, N, device="cuda") - 0.5).to(torch.bfloat16),
                          torch.empty(M, N, device="cuda", dtype=torch.bfloat16)), (M * K + K * N + M * N) * 2,
               max_sets=16)
n = len(rot.sets)
d = alcop.gemm_desc(M, N, K)
out = []
for tk in (32, 64, 128):
    for st in range(2, 17):
        s = alcop.make_schedule(tileN=tn, tileK=tk, n_stage=st, cta_group=cg)
        try:
            alcop.validate(d, s)
        except alcop.AlcopError:
            continue
        ms = time_graph(lambda i: alcop.matmul(rot.sets[i % n][0], rot.sets[i % n][1], s, out=rot.sets[i % n][2]),
                        iters=4 * n, reps_per_graph=n)
        out.append((tk, st, round(2.0 * M * N * K / ms / 1e9, 1)))
print(json.dumps({"shape": [M, N, K], "tileN": tn, "cta_group": cg, "tk_st_tflops": out}))
