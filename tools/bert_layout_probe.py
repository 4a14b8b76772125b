"""BERT GEMMs with the weight in the reference layout B[K, N] against the
nn.Linear layout B[N, K] (K-major: no over-fetch of the CTA pair's 96-column
halves, one more ring stage), per schedule; cuBLAS (torch.matmul) beside.
Measurement tool: python tools/bert_layout_probe.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2210_16691_b200 as alcop
from paper_2210_16691_b200.timing import Rotating, time_graph

out = {}
for name, M, N, K in (("qkv", 4096, 2304, 768), ("o", 4096, 768, 768), ("ffn1", 4096, 3072, 768),
                      ("ffn2", 4096, 768, 3072)):
    row = {}
    for lay in ("KN", "NK"):
        bl = alcop.B_KN if lay == "KN" else alcop.B_NK

        def mk(i):
            A = (torch.rand(M, K, device="cuda") - 0.5).to(torch.bfloat16)
            B = (torch.rand((K, N) if lay == "KN" else (N, K), device="cuda") - 0.5).to(torch.bfloat16)
            return A, B, torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        rot = Rotating(mk, (M * K + K * N + M * N) * 2, max_sets=16)
        nr = len(rot.sets)
        d = alcop.gemm_desc(M, N, K, 1, alcop.BF16, alcop.BF16, bl)
        cands = [("pick", alcop.choose_schedule(d))]
        for cg in (1, 2):
            for tn in (192, 256):
                for st in (4, 5, 6, 7, 8):
                    cands.append(("cg%d_%d_s%d" % (cg, tn, st),
                                  alcop.make_schedule(tileN=tn, tileK=64, n_stage=st, cta_group=cg)))
        best = None
        for cname, s in cands:
            try:
                alcop.validate(d, s)
                ms = time_graph(lambda i: alcop.matmul(rot.sets[i % nr][0], rot.sets[i % nr][1], s,
                                                       b_layout=bl, out=rot.sets[i % nr][2]),
                                iters=8 * nr, warmup=2, reps_per_graph=nr)
            except alcop.AlcopError:
                continue
            tf = round(2.0 * M * N * K / ms / 1e9, 1)
            if cname == "pick":
                row[lay + "_pick"] = [tf, str(s)]
            if best is None or tf > best[0]:
                best = [tf, cname]
        row[lay + "_best"] = best
        if lay == "KN":
            ms = time_graph(lambda i: torch.matmul(rot.sets[i % nr][0], rot.sets[i % nr][1], out=rot.sets[i % nr][2]),
                            iters=8 * nr, warmup=2, reps_per_graph=nr)
            row["cublas"] = round(2.0 * M * N * K / ms / 1e9, 1)
        del rot
    out[name] = row
    print(name, json.dumps(row), flush=True)
