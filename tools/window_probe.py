"""Window-mode conv (csrc/stem_sm100.cu, C = 64 stride 1) against the im2col
kernel on ResNet-50 l1 3x3 (56x56x64 -> 64, batch 256) and smaller maps:
per-schedule times.  Usage: python tools/window_probe.py [batch]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2210_16691_b200 as alcop
from paper_2210_16691_b200.timing import time_graph

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
out = {}
for H, K in ((56, 64), (28, 64), (14, 64)):
    X = (torch.rand((n, H, H, 64), device="cuda") - 0.5).to(torch.bfloat16)
    W = (torch.rand((K, 3, 3, 64), device="cuda") - 0.5).to(torch.bfloat16)
    Y = torch.empty((n, H, H, K), device="cuda", dtype=torch.bfloat16)
    fl = 2.0 * n * H * H * K * 9 * 64
    row = {}
    d = alcop.conv_desc(n, H, H, 64, K, 3, 3, (1, 1), (1, 1), alcop.BF16, alcop.BF16)
    pick = alcop.choose_conv_schedule(d)
    row["pick"] = pick.as_dict()
    cands = [("win_s%d_a%d" % (st, a), alcop.make_schedule(tileN=K, tileK=64, n_stage=st, n_stage_inner=a, mode=1))
             for st in (2, 3, 4) for a in (2, 4)]
    cands += [("im2col_%d_s%d" % (tn, st), alcop.make_schedule(tileN=tn, tileK=64, n_stage=st, n_stage_inner=2, mode=0))
              for tn, st in ((64, 8), (128, 6))]
    for name, s in cands:
        try:
            ms = time_graph(lambda i: alcop.conv2d(X, W, (1, 1), (1, 1), sched=s, out=Y), iters=10, warmup=3)
        except alcop.AlcopError as e:
            row[name] = str(e)[:60]
            continue
        row[name] = {"us": round(ms * 1e3, 1), "tflops": round(fl / ms / 1e9, 1)}
    out["%dx%d_k%d" % (H, H, K)] = row
    del X, W, Y
print(json.dumps(out))
