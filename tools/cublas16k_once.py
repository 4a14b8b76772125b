import torch
n=16384
A=(torch.rand(n,n,device='cuda')-0.5).bfloat16(); B=(torch.rand(n,n,device='cuda')-0.5).bfloat16(); C=torch.empty(n,n,device='cuda',dtype=torch.bfloat16)
torch.matmul(A,B,out=C); torch.cuda.synchronize()
torch.cuda.profiler.start(); torch.matmul(A,B,out=C); torch.cuda.synchronize(); torch.cuda.profiler.stop()
