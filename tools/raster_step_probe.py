"""The headline step (C5 squares 4096..16384, one CUDA graph of four launches
with the model's 256x512 pair schedule) in the sustained regime (~1.5 s of
steps per setting) for several raster-group sizes of the 16384 / 12288 squares
(schedule.raster; 0 = the library's auto group).  Fewer distinct A-row and
B-column panels in flight = fewer HBM re-reads = less power under the cap.
Measurement tool: python tools/raster_step_probe.py [r1 r2 ...]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2210_16691_b200 as alcop
from paper_2210_16691_b200 import workloads as W

rasters = [int(a) for a in sys.argv[1:]] or [0, 2, 4, 8, 16, 32]
bufs = {}
for n in W.SQUARES:
    bufs[n] = ((torch.rand(n, n, device="cuda") - 0.5).to(torch.bfloat16),
               (torch.rand(n, n, device="cuda") - 0.5).to(torch.bfloat16),
               torch.empty(n, n, device="cuda", dtype=torch.bfloat16))
flops = sum(2.0 * n ** 3 for n in W.SQUARES)
out = {}
for r in rasters:
    scheds = {}
    for n in W.SQUARES:
        s = W.square_schedule(alcop, n, n)
        if n >= 12288:
            s.raster = r
        scheds[n] = s
    g = torch.cuda.CUDAGraph()
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        for n in W.SQUARES:
            alcop.matmul(*bufs[n][:2], scheds[n], out=bufs[n][2])
    torch.cuda.synchronize()
    with torch.cuda.graph(g):
        for n in W.SQUARES:
            alcop.matmul(*bufs[n][:2], scheds[n], out=bufs[n][2])
    for _ in range(20):
        g.replay()
    torch.cuda.synchronize()
    t0 = time.time()
    steps = 0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    while time.time() - t0 < 1.5:
        for _ in range(10):
            g.replay()
        steps += 10
        torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    out[r] = {"ms_per_step": round(ms, 3), "tflops": round(flops / ms / 1e9, 1)}
    print(r, out[r], flush=True)
print(json.dumps(out))
