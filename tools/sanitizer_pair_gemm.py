"""compute-sanitizer case (measurement tool): one CTA-pair GEMM, exact against the oracle."""
import sys; sys.path.insert(0, '.')
import torch, numpy as np
import paper_2210_16691_b200 as alcop
from oracle import coracle
from oracle.splitmix import gemm_inputs
a, b = gemm_inputs(512, 512, 256, seed=5)
C = alcop.matmul(torch.from_numpy(a).to(torch.bfloat16).cuda(), torch.from_numpy(b).to(torch.bfloat16).cuda(),
                 alcop.make_schedule(tileN=256, tileK=64, n_stage=4, cta_group=2), out_dtype=torch.float32)
torch.cuda.synchronize()
print("pair gemm", np.array_equal(C.cpu().numpy().astype(np.int64), coracle.gemm_i64(a, b)))
