"""Where the time between the step's kernels goes (measurement tool): the four
GEMMs PDL-chained as direct launches, each with its own globaltimer stamp
buffer (alcop_debug_set_stamps before each launch); prints per kernel the
first CTA start, mean setup-done, mean first-accumulator (epilogue start),
last CTA end, relative to the first kernel's first CTA start (us)."""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2210_16691_b200 as alcop
from bench import BERT_GEMMS

lib = alcop.load_library()
lib.alcop_debug_set_stamps.argtypes = [ctypes.c_void_p]
S = alcop.make_schedule
picks = [S(256, 64, 4), S(192, 64, 5), S(256, 64, 6, cta_group=2), S(192, 64, 5)]
if len(sys.argv) > 1 and sys.argv[1] == "single":
    picks[2] = S(256, 64, 4)
sets = [[((torch.rand(M, K, device="cuda") - 0.5).to(torch.bfloat16),
          (torch.rand(K, N, device="cuda") - 0.5).to(torch.bfloat16),
          torch.empty(M, N, device="cuda", dtype=torch.bfloat16)) for _, M, N, K in BERT_GEMMS] for _ in range(3)]
bufs = [torch.zeros(148 * 8 + 256, dtype=torch.int64, device="cuda") for _ in BERT_GEMMS]
# capture one graph per input set with a stamp buffer per launch (the stamp
# pointer is a kernel parameter, so it is captured), replay, read the stamps
graphs = []
for i in range(3):
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        for j, ((A, B, C), s) in enumerate(zip(sets[i], picks)):  # warm-up outside capture
            alcop.matmul(A, B, s, out=C)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for j, ((A, B, C), s) in enumerate(zip(sets[i], picks)):
            lib.alcop_debug_set_stamps(ctypes.c_void_p(bufs[j].data_ptr()))
            alcop.matmul(A, B, s, out=C)
        lib.alcop_debug_set_stamps(None)
    graphs.append(g)
res = []
for it in range(12):
    graphs[it % 3].replay()  # back-to-back replays: the previous step's tail is in flight
    if it < 6 or it % 3 != 2:
        continue
    torch.cuda.synchronize()
    t = [b[:148 * 8].view(148, 8).cpu().numpy().astype(np.int64) for b in bufs]
    t0 = min(x[x[:, 0] > 0, 0].min() for x in t)
    row = []
    for x in t:
        x = x[x[:, 0] > 0]
        row.append({"start_first": (x[:, 0].min() - t0) / 1e3, "setup_mean": (x[:, 1].mean() - t0) / 1e3,
                    "epi_first_mean": (x[:, 5][x[:, 5] > 0].mean() - t0) / 1e3 if (x[:, 5] > 0).any() else None,
                    "end_last": (x[:, 7].max() - t0) / 1e3, "end_mean": (x[:, 7].mean() - t0) / 1e3})
    res.append(row)
avg = [{k: round(float(np.mean([r[j][k] for r in res if r[j][k] is not None])), 2) for k in res[0][j]}
       for j in range(len(BERT_GEMMS))]
for (name, *_), a in zip(BERT_GEMMS, avg):
    print(name, json.dumps(a))
