"""cta_group 2 with tileN 192 on the BERT shapes vs the 1-CTA schedules and cuBLAS."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2210_16691_b200 as alcop
from paper_2210_16691_b200.timing import Rotating, time_graph


def main():
    for M, N, K in [(4096, 768, 3072), (4096, 768, 768), (4096, 3072, 768), (8192, 8192, 8192)]:
        def mk(i):
            A = (torch.rand(M, K, device="cuda") - 0.5).to(torch.bfloat16)
            B = (torch.rand(K, N, device="cuda") - 0.5).to(torch.bfloat16)
            return A, B, torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        rot = Rotating(mk, (M * K + K * N + M * N) * 2, max_sets=16)
        n = len(rot.sets)
        iters = max(n, 20 * n if M * N * K < 2 ** 33 else 2 * n)
        flops = 2.0 * M * N * K
        ref = torch.matmul(rot.sets[0][0], rot.sets[0][1])
        out = {"shape": [M, N, K]}
        for cg, tn, tk, st in [(1, 192, 64, 4), (2, 192, 64, 4), (2, 192, 64, 5), (2, 192, 64, 6), (2, 192, 64, 7),
                               (2, 192, 128, 3), (2, 256, 64, 6), (2, 128, 64, 6)]:
            s = alcop.make_schedule(tileN=tn, tileK=tk, n_stage=st, cta_group=cg)
            try:
                ms = time_graph(lambda i: alcop.matmul(rot.sets[i % n][0], rot.sets[i % n][1], s,
                                                       out=rot.sets[i % n][2]), iters=iters, reps_per_graph=n)
            except alcop.AlcopError as e:
                out["cg%d_%d_%d_s%d" % (cg, tn, tk, st)] = str(e)[:40]
                continue
            ok = bool(torch.equal(rot.sets[0][2], ref))
            out["cg%d_%d_%d_s%d" % (cg, tn, tk, st)] = round(flops / ms / 1e9, 1) if ok else "MISMATCH"
        ms = time_graph(lambda i: torch.matmul(rot.sets[i % n][0], rot.sets[i % n][1], out=rot.sets[i % n][2]),
                        iters=iters, reps_per_graph=n)
        out["cublas"] = round(flops / ms / 1e9, 1)
        out["model"] = repr(alcop.choose_schedule(alcop.gemm_desc(M, N, K)))
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
