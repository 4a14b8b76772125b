"""One conv1 stem launch (for ncu): python tools/conv1_once.py [batch] [stages]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2210_16691_b200 as alcop

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32
stg = int(sys.argv[2]) if len(sys.argv) > 2 else 4
H, C, Cs, K, R, st, pd = 224, 3, 8, 64, 7, 2, 3
P = (H + 2 * pd - R) // st + 1
Xh = torch.zeros((n, H + 2 * pd, H + 2 * pd, Cs), device="cuda", dtype=torch.bfloat16)
Xh[:, pd:pd + H, pd:pd + H, :C] = (torch.rand((n, H, H, C), device="cuda") - 0.5).to(torch.bfloat16)
Wf = torch.zeros((K, R, R, Cs), device="cuda", dtype=torch.bfloat16)
Wf[..., :C] = (torch.rand((K, R, R, C), device="cuda") - 0.5).to(torch.bfloat16)
Y = torch.empty((n, P, P, K), device="cuda", dtype=torch.bfloat16)
s = alcop.make_schedule(tileN=64, tileK=64, n_stage=stg, n_stage_inner=2)
for _ in range(3):
    alcop.conv2d(Xh, Wf, (st, st), (pd, pd), sched=s, out=Y, x_halo=True)
torch.cuda.synchronize()
X = Xh[:, pd:pd + H, pd:pd + H, :].contiguous()
Y2 = torch.empty_like(Y)
alcop.conv2d(X, Wf, (st, st), (pd, pd), sched=s, out=Y2)
ref = torch.nn.functional.conv2d(X.permute(0, 3, 1, 2).float(), Wf.permute(0, 3, 1, 2).float(), stride=st,
                                 padding=pd).permute(0, 2, 3, 1)
for name, y in (("stem", Y), ("im2col8", Y2)):
    err = ((y.float() - ref).abs().max() / ref.abs().max()).item()
    print(name, "max rel err vs fp32 torch conv", err)
