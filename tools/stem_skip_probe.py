"""Stem kernel (csrc/stem_sm100.cu) with parts of its pipeline switched off
(ALCOP_STEM_SKIP bits: 1 no MMA, 2 no window load, 4 no store), to find
which stage sets the per-tile time.  Measurement only: skipped runs produce
wrong outputs, so the switches exist only in a probe build:
    ALCOP_BUILD_LIB=$PWD/paper_2210_16691_b200/libalcop_probe.so ALCOP_NVCC_EXTRA=-DSTEM_PROBE \
        python -m paper_2210_16691_b200._build
    ALCOP_LIB=paper_2210_16691_b200/libalcop_probe.so ALCOP_STEM_SKIP=<bits> python tools/stem_skip_probe.py <bits>"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2210_16691_b200 as alcop
from paper_2210_16691_b200.timing import time_graph

n = int(sys.argv[2]) if len(sys.argv) > 2 else 256
X = (torch.rand((n, 224, 224, 4), device="cuda") - 0.5).to(torch.bfloat16)
W = (torch.rand((64, 7, 7, 4), device="cuda") - 0.5).to(torch.bfloat16)
Y = torch.empty((n, 112, 112, 64), device="cuda", dtype=torch.bfloat16)
out = {"skip": os.environ.get("ALCOP_STEM_SKIP", "0")}
for stg, inn in ((8, 4), (8, 8), (10, 4), (10, 8), (6, 2), (12, 4)):
    s = alcop.make_schedule(tileN=64, tileK=64, n_stage=stg, n_stage_inner=inn)
    for ctas in (0,):
        s.num_ctas = ctas
        try:
            ms = time_graph(lambda i: alcop.conv2d(X, W, (2, 2), (3, 3), sched=s, out=Y), iters=10, warmup=3)
        except alcop.AlcopError as e:
            out["s%d_a%d_g%d" % (stg, inn, ctas)] = str(e)
            continue
        out["s%d_a%d_g%d" % (stg, inn, ctas)] = {"us": round(ms * 1e3, 1),
                                                  "us_per_tile_per_cta": round(ms * 1e3 / (n * 112 / (ctas or 148)), 3)}
print(json.dumps(out))
