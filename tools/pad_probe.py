import json, os, sys
sys.path.insert(0, '/root/repo')
import torch
import paper_2210_16691_b200 as alcop
from paper_2210_16691_b200.timing import Rotating, time_graph
res = {}
for name, (M, N, K) in (("ffn2", (4096, 768, 3072)), ("o", (4096, 768, 768))):
    rot = Rotating(lambda i: ((torch.rand(M, K, device="cuda") - 0.5).to(torch.bfloat16),
                              (torch.rand(K, N, device="cuda") - 0.5).to(torch.bfloat16),
                              torch.empty(M, N, device="cuda", dtype=torch.bfloat16)), (M * K + K * N + M * N) * 2, max_sets=16)
    nr = len(rot.sets)
    d = alcop.gemm_desc(M, N, K)
    for st in (5, 6, 7):
        s = alcop.make_schedule(tileN=192, tileK=64, n_stage=st, cta_group=2)
        try:
            alcop.validate(d, s)
        except alcop.AlcopError as e:
            res["%s_s%d" % (name, st)] = str(e)[:40]; continue
        ms = time_graph(lambda i: alcop.matmul(rot.sets[i % nr][0], rot.sets[i % nr][1], s, out=rot.sets[i % nr][2]), iters=4 * nr, reps_per_graph=nr)
        res["%s_s%d" % (name, st)] = round(2.0 * M * N * K / ms / 1e9, 1)
    s = alcop.make_schedule(tileN=192, tileK=64, n_stage=5)
    ms = time_graph(lambda i: alcop.matmul(rot.sets[i % nr][0], rot.sets[i % nr][1], s, out=rot.sets[i % nr][2]), iters=4 * nr, reps_per_graph=nr)
    res["%s_single192s5" % name] = round(2.0 * M * N * K / ms / 1e9, 1)
print(json.dumps({"pad": os.environ.get("ALCOP_PAIR_B_PAD", "1"), **res}))
