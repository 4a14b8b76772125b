"""Window conv kernel on CTA pairs (cta_group 2) against one CTA per tile:
ResNet-50 l1 3x3 (56x56x64 -> 64, resident filter) and l2 3x3 (28x28x128 ->
128, streamed filter) at batch 256, per-schedule times over rotating x / y
copies (> 2x L2).  Usage: python tools/window_pair_probe.py [batch]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2210_16691_b200 as alcop
from paper_2210_16691_b200.timing import Rotating, time_graph

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
out = {}
for name, H, C, K in (("l1_3x3", 56, 64, 64), ("l2_3x3", 28, 128, 128)):
    rot = Rotating(lambda i: ((torch.rand((n, H, H, C), device="cuda") - 0.5).to(torch.bfloat16),
                              torch.empty((n, H, H, K), device="cuda", dtype=torch.bfloat16)),
                   n * H * H * (C + K) * 2, max_sets=4)
    W = (torch.rand((K, 3, 3, C), device="cuda") - 0.5).to(torch.bfloat16)
    nr = len(rot.sets)
    fl = 2.0 * n * H * H * K * 9 * C
    row = {}
    d = alcop.conv_desc(n, H, H, C, K, 3, 3, (1, 1), (1, 1), alcop.BF16, alcop.BF16)
    row["pick"] = alcop.choose_conv_schedule(d).as_dict()
    cands = []
    for cg in (1, 2):
        if C == 64:
            for st, a in ((2, 2), (3, 2), (4, 2), (2, 4), (4, 4), (3, 3)):
                cands.append(("cg%d_s%d_a%d" % (cg, st, a),
                              alcop.make_schedule(tileN=K, tileK=64, n_stage=st, n_stage_inner=a, cta_group=cg)))
        else:
            for tk in (64, 192):
                for sa, sb in ((2, 2), (2, 3), (2, 4), (1, 4), (3, 3), (2, 6)):
                    cands.append(("cg%d_tk%d_a%d_b%d" % (cg, tk, sa, sb),
                                  alcop.make_schedule(tileN=K, tileK=tk, n_stage=sa, n_stage_B=sb, n_stage_inner=2,
                                                      cta_group=cg)))
    res = {}
    for rnd in range(3):  # round-robin rounds, median
        for cname, s in cands:
            try:
                ms = time_graph(lambda i: alcop.conv2d(rot.sets[i % nr][0], W, (1, 1), (1, 1), sched=s,
                                                       out=rot.sets[i % nr][1]),
                                iters=max(2 * nr, 8), warmup=3, reps_per_graph=nr)
            except alcop.AlcopError as e:
                row[cname] = str(e)[:60]
                continue
            res.setdefault(cname, []).append(ms)
    for cname, v in res.items():
        ms = sorted(v)[len(v) // 2]
        row[cname] = {"us": round(ms * 1e3, 1), "tflops": round(fl / ms / 1e9, 1)}
    out[name] = row
    del rot, W
print(json.dumps(out))
