"""The layer step (four PDL-chained launches) under different schedule mixes
(measurement tool): is the inter-kernel gap a property of mixing single-CTA
and CTA-pair kernels?"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2210_16691_b200 as alcop
from bench import BERT_GEMMS
from paper_2210_16691_b200.timing import time_graph

nsets = 3
sets = [[((torch.rand(M, K, device="cuda") - 0.5).to(torch.bfloat16),
          (torch.rand(K, N, device="cuda") - 0.5).to(torch.bfloat16),
          torch.empty(M, N, device="cuda", dtype=torch.bfloat16)) for _, M, N, K in BERT_GEMMS] for _ in range(nsets)]
flops = sum(2.0 * M * N * K for _, M, N, K in BERT_GEMMS)
S = alcop.make_schedule
mixes = {
    "tuned": [S(256, 64, 4), S(192, 64, 5), S(256, 64, 6, cta_group=2), S(192, 64, 5)],
    "all_single": [S(256, 64, 4), S(192, 64, 5), S(256, 64, 4), S(192, 64, 5)],
    "all_pair": [S(256, 64, 6, cta_group=2), S(192, 64, 6, cta_group=2), S(256, 64, 6, cta_group=2),
                 S(192, 64, 6, cta_group=2)],
}
res = {}
for name, picks in mixes.items():
    def four(i, picks=picks):
        for (A, B, C), s in zip(sets[i % nsets], picks):
            alcop.matmul(A, B, s, out=C)
    ms = [time_graph(four, iters=300, reps_per_graph=nsets) for _ in range(2)]
    iso = []
    for (A, B, C), s in zip(sets[0], picks):
        iso.append(time_graph(lambda i, A=A, B=B, C=C, s=s: alcop.matmul(A, B, s, out=C), iters=60) * 1e3)
    res[name] = {"step_us": [round(m * 1e3, 2) for m in ms], "sum_isolated_warm_us": round(sum(iso), 2),
                 "isolated_us": [round(x, 2) for x in iso]}
print(json.dumps(res))
