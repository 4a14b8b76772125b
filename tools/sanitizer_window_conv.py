"""compute-sanitizer case (measurement tool): small window convs on CTA pairs and one CTA per tile,
exact against the oracle.  compute-sanitizer --tool memcheck|racecheck python tools/sanitizer_window_conv.py"""
import sys; sys.path.insert(0, '.')
import torch, numpy as np
import paper_2210_16691_b200 as alcop
from oracle import coracle
from oracle.splitmix import random_tensor
for (N,H,W,C,K), sch in (((1,28,28,64,64), dict(tileN=64,tileK=64,n_stage=2,n_stage_inner=2,cta_group=2)),
                         ((1,14,14,128,128), dict(tileN=128,tileK=64,n_stage=2,n_stage_B=3,n_stage_inner=2,cta_group=2)),
                         ((1,28,28,64,64), dict(tileN=64,tileK=64,n_stage=3,n_stage_inner=2,cta_group=1))):
    x = random_tensor(N*H*W*C, 1).reshape(N,H,W,C); w = random_tensor(K*9*C, 2).reshape(K,3,3,C)
    ref = coracle.conv2d(coracle.to_dtype(x.astype(np.float32),"bf16"), coracle.to_dtype(w.astype(np.float32),"bf16"), (1,1),(1,1),"bf16","f32")
    s = alcop.make_schedule(**sch); s.num_ctas = 4
    Y = alcop.conv2d(torch.from_numpy(x).to(torch.bfloat16).cuda(), torch.from_numpy(w).to(torch.bfloat16).cuda(), (1,1),(1,1), sched=s, out_dtype=torch.float32)
    torch.cuda.synchronize()
    print((N,H,W,C,K), sch.get('cta_group'), np.array_equal(Y.cpu().numpy(), ref))
