"""KN (MN-major B) vs NK (K-major B) at a few schedules (debug probe)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2210_16691_b200 as alcop
from paper_2210_16691_b200.timing import time_fn
M = N = K = 8192
A = (torch.rand(M, K, device="cuda") - 0.5).to(torch.bfloat16)
Bkn = (torch.rand(K, N, device="cuda") - 0.5).to(torch.bfloat16)
Bnk = Bkn.t().contiguous()
C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
for tN, tK, st in [(64, 32, 8), (64, 64, 8), (128, 64, 4), (256, 64, 4), (256, 32, 6), (128, 128, 3)]:
    s = alcop.make_schedule(tileN=tN, tileK=tK, n_stage=st)
    r = []
    for lay, B in ((alcop.B_KN, Bkn), (alcop.B_NK, Bnk)):
        ms = time_fn(lambda: alcop.matmul(A, B, s, out=C, b_layout=lay), iters=5, warmup=2)
        r.append(round(2 * M * N * K / ms / 1e9))
    print(tN, tK, st, "KN", r[0], "NK", r[1], flush=True)
