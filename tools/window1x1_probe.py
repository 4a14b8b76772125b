"""1x1 C=64 convs (ResNet-50 l1_1x1_64_64 / l1_1x1_64_256, batch 256): the
window (resident-filter) kernel (ALCOP_WINDOW_1X1=1) against the generic
implicit-GEMM kernel's model pick.  Measurement only."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2210_16691_b200 as alcop
from paper_2210_16691_b200 import workloads as Wl
from paper_2210_16691_b200.timing import time_graph

n = 256
out = {"window_1x1": os.environ.get("ALCOP_WINDOW_1X1", "0")}
for K in (64, 256):
    X = (torch.rand((n, 56, 56, 64), device="cuda") - 0.5).to(torch.bfloat16)
    W = (torch.rand((K, 1, 1, 64), device="cuda") - 0.5).to(torch.bfloat16)
    Y = torch.empty((n, 56, 56, K), device="cuda", dtype=torch.bfloat16)
    byts = X.numel() * 2 + Y.numel() * 2
    d = alcop.conv_desc(n, 56, 56, 64, K, 1, 1, (1, 1), (0, 0), alcop.BF16, alcop.BF16)
    row = {}
    cands = [("pick", alcop.choose_conv_schedule(d))]
    if os.environ.get("ALCOP_WINDOW_1X1") == "1":
        cands += [("win_s%d_a%d" % (st, a), alcop.make_schedule(tileN=K, tileK=64, n_stage=st, n_stage_inner=a))
                  for st, a in ((2, 2), (4, 2), (6, 2), (4, 1))]
    for name, s in cands:
        try:
            ms = time_graph(lambda i: alcop.conv2d(X, W, (1, 1), (0, 0), sched=s, out=Y), iters=10, warmup=3)
        except alcop.AlcopError as e:
            row[name] = str(e)[:60]
            continue
        row[name] = {"us": round(ms * 1e3, 1), "GBps": round(byts / ms / 1e6, 1), "sched": str(s)}
    out["k%d" % K] = row
print(json.dumps(out))
