"""Prints TFLOP/s of a fixed list of (shape, schedule) points — run under two
builds (ALCOP_LIB=...) to A/B a kernel change."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2210_16691_b200 as alcop
from paper_2210_16691_b200.timing import Rotating, time_graph
POINTS = [((8192, 8192, 8192), (256, 64, 4, 2)), ((8192, 8192, 8192), (256, 64, 6, 2)), ((4096, 4096, 4096), (256, 64, 4, 2)),
          ((4096, 768, 768), (256, 64, 4, 2)), ((4096, 768, 768), (128, 64, 6, 2)), ((4096, 3072, 768), (256, 64, 4, 2)),
          ((4096, 768, 3072), (256, 64, 4, 2)), ((4096, 768, 3072), (128, 64, 6, 2)), ((16384, 4096, 4096), (256, 64, 4, 2)),
          ((8192, 8192, 8192), (64, 32, 8)), ((8192, 8192, 8192), (128, 64, 4)), ((8192, 8192, 8192), (256, 64, 4)),
          ((8192, 8192, 8192), (256, 128, 2)), ((4096, 4096, 4096), (256, 64, 4)),
          ((4096, 768, 768), (256, 64, 4)), ((4096, 768, 768), (128, 64, 4)), ((4096, 768, 768), (64, 64, 6)),
          ((4096, 3072, 768), (256, 64, 4)), ((4096, 768, 3072), (256, 64, 4)), ((4096, 768, 3072), (128, 128, 3))]
tag = os.path.basename(alcop.LIB_PATH)
for (M, N, K), cfg in POINTS:
    tN, tK, st = cfg[:3]
    cg = cfg[3] if len(cfg) > 3 else 1
    mk = lambda i: ((torch.rand(M, K, device="cuda") - .5).to(torch.bfloat16), (torch.rand(K, N, device="cuda") - .5).to(torch.bfloat16), torch.empty(M, N, device="cuda", dtype=torch.bfloat16))
    rot = Rotating(mk, (M * K + K * N + M * N) * 2, max_sets=6)
    s = alcop.make_schedule(tileN=tN, tileK=tK, n_stage=st, cta_group=cg)
    def f(i):
        A, B, C = rot.next()
        alcop.matmul(A, B, s, out=C)
    ms = time_graph(f, iters=5 if M * N * K > 1e11 else 50, warmup=3)
    print("%-22s %-16s %dx%dx%d s%d %7.1f TF" % (tag, "%dx%dx%d" % (M, N, K), 128 * cg, tN, tK, st, 2 * M * N * K / ms / 1e9), flush=True)
