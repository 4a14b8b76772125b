"""Implicit-GEMM conv layers (C % 64 == 0, N >= 256) on CTA pairs vs single
CTAs (batch 256, rotating inputs > 2x L2, round-robin rounds, median).
Measurement tool: python tools/conv_pair_probe.py"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2210_16691_b200 as alcop
from paper_2210_16691_b200 import workloads as W
from paper_2210_16691_b200.timing import time_graph

names = sys.argv[1:] or ["l2_ds_256_512", "l3_3x3s2_256", "l3_3x3_256", "l3_ds_512_1024", "l4_3x3s2_512",
                         "l4_3x3_512", "l4_ds_1024_2048", "l2_3x3s2_128"]
out = {}
for name in names:
    L = [c for c in W.CONV_LAYERS if c.name == name][0]
    n = 256
    nsets = int(min(8, max(1, -(-2 * 126 * 2 ** 20 // ((n * L.H * L.H * L.Cs + n * L.P * L.P * L.K) * 2)))))
    Xs = [(torch.rand((n, L.H, L.H, L.Cs), device="cuda") - 0.5).to(torch.bfloat16) for _ in range(nsets)]
    Wf = (torch.rand((L.K, L.R, L.R, L.Cs), device="cuda") - 0.5).to(torch.bfloat16)
    Ys = [torch.empty((n, L.P, L.P, L.K), device="cuda", dtype=torch.bfloat16) for _ in range(nsets)]
    cands = {"single_256_s4": alcop.make_schedule(tileN=256, tileK=64, n_stage=4),
             "single_192_s5": alcop.make_schedule(tileN=192, tileK=64, n_stage=5),
             "single_128_s6": alcop.make_schedule(tileN=128, tileK=64, n_stage=6),
             "pair_256_s6": alcop.make_schedule(tileN=256, tileK=64, n_stage=6, cta_group=2),
             "pair_192_s7": alcop.make_schedule(tileN=192, tileK=64, n_stage=7, cta_group=2),
             "pair_128_s8": alcop.make_schedule(tileN=128, tileK=64, n_stage=8, cta_group=2),
             "model": W.conv_schedule(alcop, L, n)}
    times = {k: [] for k in cands}
    for _ in range(3):
        for k, s in cands.items():
            fn = lambda i, s=s: alcop.conv2d(Xs[i % nsets], Wf, (L.stride,) * 2, (L.pad,) * 2, sched=s,
                                            out=Ys[i % nsets])
            try:
                times[k].append(time_graph(fn, iters=max(nsets, 12 // nsets * nsets), warmup=1))
            except alcop.AlcopError as e:
                times[k] = str(e)[:50]
    row = {k: (round(L.flops(n) / statistics.median(v) / 1e9, 1) if isinstance(v, list) else v)
           for k, v in times.items()}
    row["model_sched"] = str(cands["model"])
    out[name] = row
    print(name, json.dumps(row), flush=True)
    del Xs, Ys, Wf
    torch.cuda.empty_cache()
