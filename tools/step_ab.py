"""The bench's layer step (four PDL-chained launches, model schedules) timed
against a given libalcop build (measurement tool): python tools/step_ab.py [lib]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2210_16691_b200 as alcop
from paper_2210_16691_b200.timing import time_graph

if len(sys.argv) > 1:
    alcop.LIB_PATH = sys.argv[1]
from bench import BERT_GEMMS  # noqa: E402

nsets = 3
sets = [[((torch.rand(M, K, device="cuda") - 0.5).to(torch.bfloat16),
          (torch.rand(K, N, device="cuda") - 0.5).to(torch.bfloat16),
          torch.empty(M, N, device="cuda", dtype=torch.bfloat16)) for _, M, N, K in BERT_GEMMS] for _ in range(nsets)]
flops = sum(2.0 * M * N * K for _, M, N, K in BERT_GEMMS)
picks = [alcop.choose_schedule(alcop.gemm_desc(M, N, K)) for _, M, N, K in BERT_GEMMS]


def four(i):
    for (A, B, C), s in zip(sets[i % nsets], picks):
        alcop.matmul(A, B, s, out=C)


res = []
for _ in range(3):
    ms = time_graph(four, iters=300, reps_per_graph=nsets)
    res.append(round(flops / ms / 1e9, 1))
print(json.dumps({"lib": alcop.LIB_PATH[-24:], "step_tflops": res, "picks": [repr(s) for s in picks]}))
