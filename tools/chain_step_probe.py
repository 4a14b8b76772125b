"""The BERT-layer step as ONE alcop_gemm_chain launch vs four launches
(measurement tool): schedules x {independent, row-block dependencies}."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2210_16691_b200 as alcop
from bench import BERT_GEMMS
from paper_2210_16691_b200.timing import time_graph

nsets = 3
sets = []
for _ in range(nsets):
    sets.append([((torch.rand(M, K, device="cuda") - 0.5).to(torch.bfloat16),
                  (torch.rand(K, N, device="cuda") - 0.5).to(torch.bfloat16),
                  torch.empty(M, N, device="cuda", dtype=torch.bfloat16)) for _, M, N, K in BERT_GEMMS])
flops = sum(2.0 * M * N * K for _, M, N, K in BERT_GEMMS)
ws = torch.empty(1 << 16, dtype=torch.uint8, device="cuda")
res = {}
for tn, tk, st in ((192, 64, 5), (256, 64, 4), (192, 128, 2), (256, 128, 2), (128, 64, 6), (128, 128, 3)):
    s = alcop.make_schedule(tileN=tn, tileK=tk, n_stage=st)
    for dep in ([0, 0, 0, 0], [0, 1, 1, 1]):
        ms = time_graph(lambda i: alcop.gemm_chain(sets[i % nsets], s, dep=dep, workspace=ws), iters=60,
                        reps_per_graph=nsets)
        res["%dx%dx%d s%d dep%d" % (128, tn, tk, st, dep[1])] = {"us": round(ms * 1e3, 2),
                                                                   "tflops": round(flops / ms / 1e9, 1)}
# four launches with the tuned per-GEMM picks, same rotating sets
picks = [alcop.choose_schedule(alcop.gemm_desc(M, N, K)) for _, M, N, K in BERT_GEMMS]


def four(i):
    for (A, B, C), s in zip(sets[i % nsets], picks):
        alcop.matmul(A, B, s, out=C)
ms = time_graph(four, iters=60, reps_per_graph=nsets)
res["four launches (model picks)"] = {"us": round(ms * 1e3, 2), "tflops": round(flops / ms / 1e9, 1)}
print(json.dumps(res, indent=0))
