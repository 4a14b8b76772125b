"""CTA 0's MMA-thread timeline of one CTA-pair GEMM launch from the
-DGEMM_TRACE build (ALCOP_LIB=paper_2210_16691_b200/libalcop_gtrace.so):
per chunk, clock64 after the full-barrier wait and after the chunk's MMAs +
commit were issued.  Measurement only.  python tools/gemm_trace.py M N K tileN tileK stages"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2210_16691_b200 as alcop

M, N, K, tn, tk, st = map(int, sys.argv[1:7])
A = (torch.rand(M, K, device="cuda") - 0.5).to(torch.bfloat16)
B = (torch.rand(K, N, device="cuda") - 0.5).to(torch.bfloat16)
C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
s = alcop.make_schedule(tileN=tn, tileK=tk, n_stage=st, cta_group=2)
alcop.matmul(A, B, s, out=C)
torch.cuda.synchronize()
