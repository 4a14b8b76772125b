"""Attention BMMs (192 x QK^T 512x512x64, PV 512x64x512): the bench's tuned
schedule at several persistent grid sizes (num_ctas) and tile widths — does a
grid that divides the tile count evenly (no partial last wave) help an
HBM-bound launch?  Rotating inputs (> 2x L2), CUDA graphs, round-robin rounds,
median.  Usage: python tools/bmm_grid_probe.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2210_16691_b200 as alcop
from paper_2210_16691_b200.timing import Rotating, time_graph

nb = 192
out = {}
for name, (M, N, K), base in (("qkt", (512, 512, 64), dict(tileN=256, tileK=64, n_stage=4)),
                              ("pv", (512, 64, 512), dict(tileN=64, tileK=128, n_stage=4))):
    rot = Rotating(lambda i: ((torch.rand((nb, M, K), device="cuda") - 0.5).to(torch.bfloat16),
                              (torch.rand((nb, K, N), device="cuda") - 0.5).to(torch.bfloat16),
                              torch.empty((nb, M, N), device="cuda", dtype=torch.bfloat16)),
                   (M * K + K * N + M * N) * 2 * nb, max_sets=16)
    nr = len(rot.sets)
    byts = (M * K + K * N + M * N) * 2 * nb
    tiles = nb * (M // 128) * ((N + base["tileN"] - 1) // base["tileN"])
    cands = {}
    for nc in (148, 144, 128, 96, 74):
        s = alcop.make_schedule(**base)
        s.num_ctas = nc
        cands["ctas%d_waves%.2f" % (nc, tiles / nc)] = s
    if name == "pv":
        for tk, st in ((64, 6), (64, 8), (128, 3), (256, 2)):
            cands["tk%d_s%d" % (tk, st)] = alcop.make_schedule(tileN=64, tileK=tk, n_stage=st)
    else:
        for tn, st in ((128, 6), (512, 2)):
            cands["tn%d_s%d" % (tn, st)] = alcop.make_schedule(tileN=tn, tileK=64, n_stage=st)
    res = {}
    for rnd in range(3):
        for cname, s in cands.items():
            try:
                ms = time_graph(lambda i: alcop.matmul(rot.sets[i % nr][0], rot.sets[i % nr][1], s,
                                                       out=rot.sets[i % nr][2]),
                                iters=8 * nr, warmup=3, reps_per_graph=nr)
            except alcop.AlcopError as e:
                res[cname] = str(e)[:50]
                continue
            res.setdefault(cname, []).append(ms)
    out[name] = {k: (v if isinstance(v, str) else {"us": round(sorted(v)[1] * 1e3, 2),
                                                   "gbs": round(byts / sorted(v)[1] / 1e6, 1)})
                 for k, v in res.items()}
    del rot
print(json.dumps(out))
