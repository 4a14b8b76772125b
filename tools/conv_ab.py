"""A/B timing of ResNet-50 conv layers against a given libalcop build
(measurement tool): python tools/conv_ab.py [path/to/libalcop.so]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2210_16691_b200 as alcop
from paper_2210_16691_b200.timing import time_graph

if len(sys.argv) > 1:
    alcop.LIB_PATH = sys.argv[1]
from bench import RESNET50_CONVS  # noqa: E402

res = {}
for (name, H, C, K, R, st, pd, rep) in RESNET50_CONVS[:6] + RESNET50_CONVS[13:14] + RESNET50_CONVS[19:20]:
    n = 256
    P, Q = alcop.conv_out_hw(H, H, R, R, (st, st), (pd, pd))
    Cs = -(-C // 8) * 8
    halo = R * Cs <= 64
    hp = pd if halo else 0
    g = alcop.gemm_desc(n * P * Q, K, R * 64 if halo else R * R * Cs, 1, alcop.BF16, alcop.BF16, alcop.B_NK)
    cs = alcop.choose_conv_schedule(alcop.conv_desc(n, H, H, C, K, R, R, (st, st), (pd, pd)))
    X = torch.zeros((n, H + 2 * hp, H + 2 * hp, Cs), device="cuda", dtype=torch.bfloat16)
    Wf = torch.zeros((K, R, R, Cs), device="cuda", dtype=torch.bfloat16)
    X[:, hp:hp + H, hp:hp + H, :C] = (torch.rand((n, H, H, C), device="cuda") - 0.5).to(torch.bfloat16)
    Wf[..., :C] = (torch.rand((K, R, R, C), device="cuda") - 0.5).to(torch.bfloat16)
    Y = torch.empty((n, P, Q, K), device="cuda", dtype=torch.bfloat16)
    ms = time_graph(lambda i: alcop.conv2d(X, Wf, (st, st), (pd, pd), sched=cs, out=Y, x_halo=halo), iters=6, warmup=2)
    res[name] = [round(2.0 * n * P * Q * K * R * R * C / (ms * 1e-3) / 1e12, 1), repr(cs)]
print(json.dumps({"lib": alcop.LIB_PATH, "layers": res}))

# BERT-layer GEMMs with fixed schedules valid in both builds
from paper_2210_16691_b200.timing import Rotating  # noqa: E402
gres = {}
for name, (M, N, K), (tn, tk, st, cg) in (("qkv", (4096, 2304, 768), (256, 64, 4, 1)),
                                          ("o", (4096, 768, 768), (192, 64, 4, 1)),
                                          ("ffn1", (4096, 3072, 768), (256, 128, 3, 2)),
                                          ("ffn2", (4096, 768, 3072), (192, 64, 4, 1))):
    rot = Rotating(lambda i: ((torch.rand(M, K, device="cuda") - 0.5).to(torch.bfloat16),
                              (torch.rand(K, N, device="cuda") - 0.5).to(torch.bfloat16),
                              torch.empty(M, N, device="cuda", dtype=torch.bfloat16)), (M * K + K * N + M * N) * 2,
                   max_sets=16)
    nr = len(rot.sets)
    s = alcop.make_schedule(tileN=tn, tileK=tk, n_stage=st, cta_group=cg)
    ms = time_graph(lambda i: alcop.matmul(rot.sets[i % nr][0], rot.sets[i % nr][1], s, out=rot.sets[i % nr][2]),
                    iters=4 * nr, reps_per_graph=nr)
    gres[name] = round(2.0 * M * N * K / ms / 1e9, 1)
print(json.dumps({"lib": alcop.LIB_PATH, "gemms": gres}))
