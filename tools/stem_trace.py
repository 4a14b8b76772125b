"""One launch of the stem kernel from the -DSTEM_TRACE build (ALCOP_LIB=
paper_2210_16691_b200/libalcop_trace.so): CTA 0's per-tile role timestamps
(tiles 40+), printed as deltas in ns.  Measurement only."""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2210_16691_b200 as alcop

n = 64
X = (torch.rand((n, 224, 224, 4), device="cuda") - 0.5).to(torch.bfloat16)
W = (torch.rand((64, 7, 7, 4), device="cuda") - 0.5).to(torch.bfloat16)
Y = torch.empty((n, 112, 112, 64), device="cuda", dtype=torch.bfloat16)
s = alcop.make_schedule(tileN=64, tileK=64, n_stage=8, n_stage_inner=4)
alcop.conv2d(X, W, (2, 2), (3, 3), sched=s, out=Y)
torch.cuda.synchronize()
