"""One ResNet-50 conv layer (l3 3x3 256->256, batch 256) and one attention
QK^T BMM (192 x 512x512x64) with the bench's model schedules, for an
`ncu --set full` capture (measurement tool; launch order: conv, bmm)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2210_16691_b200 as alcop

n, H, C, K, R = 256, 14, 256, 256, 3
P, Q = alcop.conv_out_hw(H, H, R, R, (1, 1), (1, 1))
g = alcop.gemm_desc(n * P * Q, K, R * R * C, 1, alcop.BF16, alcop.BF16, alcop.B_NK)
cs = alcop.choose_conv_schedule(alcop.conv_desc(n, H, H, C, K, R, R, (1, 1), (1, 1)))
X = (torch.rand((n, H, H, C), device="cuda") - 0.5).to(torch.bfloat16)
W = (torch.rand((K, R, R, C), device="cuda") - 0.5).to(torch.bfloat16)
Y = torch.empty((n, P, Q, K), device="cuda", dtype=torch.bfloat16)
A = (torch.rand((192, 512, 64), device="cuda") - 0.5).to(torch.bfloat16)
B = (torch.rand((192, 64, 512), device="cuda") - 0.5).to(torch.bfloat16)
Cb = torch.empty((192, 512, 512), device="cuda", dtype=torch.bfloat16)
sb = alcop.choose_schedule(alcop.gemm_desc(512, 512, 64, 192))
for _ in range(3):
    alcop.conv2d(X, W, (1, 1), (1, 1), sched=cs, out=Y)
    alcop.matmul(A, B, sb, out=Cb)
torch.cuda.synchronize()
print("conv", cs, "bmm", sb)
