"""A/B of CTA-pair GEMM schedules against a given libalcop build
(measurement tool): python tools/pair_ab.py [path/to/libalcop.so]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2210_16691_b200 as alcop
from paper_2210_16691_b200.timing import Rotating, time_graph

if len(sys.argv) > 1:
    alcop.LIB_PATH = sys.argv[1]
CONV1X1 = (("l3_1x1_pair256s6", (50176, 1024, 256), (256, 64, 6, 2)),
           ("l3_1x1_single256s3", (50176, 1024, 256), (256, 64, 3, 1)),
           ("l2_1x1_pair256s6", (200704, 512, 128), (256, 64, 6, 2)),
           ("l2_1x1_single256s3", (200704, 512, 128), (256, 64, 3, 1)),
           ("l4_1x1_pair256s6", (12544, 2048, 512), (256, 64, 6, 2)),
           ("l4_1x1_single192s5", (12544, 2048, 512), (192, 64, 5, 1)),
           ("l1_1x1_pair256s6", (802816, 256, 64), (256, 64, 6, 2)),
           ("l1_1x1_single128s4", (802816, 256, 64), (128, 64, 4, 1)),
           ("l3_1x1_1024_256_pair256s6", (50176, 256, 1024), (256, 64, 6, 2)))
res = {}
cases = (("ffn1_64s6", (4096, 3072, 768), (256, 64, 6, 2)),
                                          ("ffn1_128s3", (4096, 3072, 768), (256, 128, 3, 2)),
                                          ("qkv_64s6", (4096, 2304, 768), (256, 64, 6, 2)),
                                          ("ffn2_192s6", (4096, 768, 3072), (192, 64, 6, 2)),
                                          ("sq8192_64s6", (8192, 8192, 8192), (256, 64, 6, 2)),
                                          ("sq8192_128s3", (8192, 8192, 8192), (256, 128, 3, 2)),
                                          ("single_ffn1_256s4", (4096, 3072, 768), (256, 64, 4, 1)),
                                          ("single_ffn2_192s5", (4096, 768, 3072), (192, 64, 5, 1)),
                                          ("single_o_192s5", (4096, 768, 768), (192, 64, 5, 1)))
if os.environ.get("PAIR_AB_SET") == "conv1x1":  # the ResNet-50 1x1 convs' GEMM views at batch 256
    cases = CONV1X1
for name, (M, N, K), (tn, tk, st, cg) in cases:
    rot = Rotating(lambda i: ((torch.rand(M, K, device="cuda") - 0.5).to(torch.bfloat16),
                              (torch.rand(K, N, device="cuda") - 0.5).to(torch.bfloat16),
                              torch.empty(M, N, device="cuda", dtype=torch.bfloat16)), (M * K + K * N + M * N) * 2,
                   max_sets=8)
    nr = len(rot.sets)
    s = alcop.make_schedule(tileN=tn, tileK=tk, n_stage=st, cta_group=cg)
    ms = time_graph(lambda i: alcop.matmul(rot.sets[i % nr][0], rot.sets[i % nr][1], s, out=rot.sets[i % nr][2]),
                    iters=max(4 * nr, 8), reps_per_graph=nr)
    res[name] = round(2.0 * M * N * K / ms / 1e9, 1)
    del rot
print(json.dumps({"lib": alcop.LIB_PATH[-24:], "pair": res}))
