"""CTA 0's MMA-thread timeline of one CTA-pair GEMM launch from the
-DGEMM_TRACE build (ALCOP_LIB=paper_2210_16691_b200/libalcop_gtrace.so):
per chunk, clock64 after the full-barrier wait and after the chunk's MMAs +
commit were issued, plus per tile the start and the
accumulator-free time.  Measurement only; --parse FILE summarises a saved run.  python tools/gemm_trace.py M N K tileN tileK stages"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2210_16691_b200 as alcop


def parse(path):
    """Per tile: clk from tile start to accumulator free, the chunks' full-wait
    times and the issue spans, relative to the first record."""
    recs = [int(l.split()[2]) for l in open(path) if l.startswith("T ")]
    base = None
    tiles = []
    for r in recs:
        v = r & ((1 << 61) - 1)
        base = v if base is None else base
        if r >> 62 & 1:
            tiles.append({"start": v - base, "acc_free": None, "chunks": []})
        elif r >> 61 & 1:
            tiles[-1]["acc_free"] = v - base
        else:
            tiles[-1]["chunks"].append(v - base)
    for t in tiles:
        w = t["chunks"][0::2]
        print("tile start %6d  acc free +%5d  chunk waits %s" % (
            t["start"], (t["acc_free"] or 0) - t["start"], [x - t["start"] for x in w]))


if sys.argv[1] == "--parse":
    parse(sys.argv[2])
    sys.exit(0)
M, N, K, tn, tk, st = map(int, sys.argv[1:7])
A = (torch.rand(M, K, device="cuda") - 0.5).to(torch.bfloat16)
B = (torch.rand(K, N, device="cuda") - 0.5).to(torch.bfloat16)
C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
s = alcop.make_schedule(tileN=tn, tileK=tk, n_stage=st, cta_group=2)
alcop.matmul(A, B, s, out=C)
torch.cuda.synchronize()
