"""Which cuBLAS kernels (tile, cluster, split) run the BERT-layer shapes —
context for the schedule space (run under ncu to see names/grids)."""
import sys
import torch

SHAPES = [(4096, 768, 768), (4096, 2304, 768), (4096, 3072, 768), (4096, 768, 3072), (8192, 8192, 8192)]
for M, N, K in SHAPES:
    A = (torch.rand(M, K, device="cuda") - 0.5).to(torch.bfloat16)
    B = (torch.rand(K, N, device="cuda") - 0.5).to(torch.bfloat16)
    for _ in range(3):
        torch.matmul(A, B)
    torch.cuda.synchronize()
