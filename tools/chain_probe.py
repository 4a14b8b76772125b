import sys, os, json
sys.path.insert(0, '/root/repo')
import torch
import paper_2210_16691_b200 as alcop
from paper_2210_16691_b200.timing import Rotating, time_graph
res = {}
for (M, N, K, reps) in ((4096, 768, 768, 4), (16384, 768, 768, 1), (4096, 768, 3072, 2), (8192, 768, 3072, 1), (4096, 3072, 768, 2), (8192, 3072, 768, 1)):
    rot = Rotating(lambda i: ((torch.rand(M, K, device="cuda") - 0.5).to(torch.bfloat16),
                              (torch.rand(K, N, device="cuda") - 0.5).to(torch.bfloat16),
                              torch.empty(M, N, device="cuda", dtype=torch.bfloat16)), (M * K + K * N + M * N) * 2, max_sets=16)
    nr = len(rot.sets)
    s = alcop.choose_schedule(alcop.gemm_desc(M, N, K))
    ms = time_graph(lambda i: alcop.matmul(rot.sets[i % nr][0], rot.sets[i % nr][1], s, out=rot.sets[i % nr][2]), iters=4 * nr, reps_per_graph=nr)
    res["%dx%dx%d" % (M, N, K)] = {"us_per_launch": round(ms * 1e3, 2), "us_for_equal_work": round(ms * 1e3 * reps, 2), "tflops": round(2.0*M*N*K/ms/1e9, 1), "sched": repr(s)}
print(json.dumps(res, indent=0))
