"""Raster-group sweep: TFLOP/s of a fixed schedule per schedule.raster value
(0 = auto), cuBLAS beside it.  Usage: python tools/raster_probe.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2210_16691_b200 as alcop
from paper_2210_16691_b200.timing import Rotating, time_graph

CASES = [((8192, 8192, 8192), dict(cta_group=2, tileN=256, tileK=64, n_stage=6)),
         ((16384, 4096, 4096), dict(cta_group=2, tileN=256, tileK=64, n_stage=6)),
         ((4096, 4096, 4096), dict(cta_group=2, tileN=256, tileK=64, n_stage=6)),
         ((4096, 3072, 768), dict(cta_group=2, tileN=256, tileK=64, n_stage=6)),
         ((4096, 768, 3072), dict(cta_group=1, tileN=192, tileK=64, n_stage=4)),
         ((8192, 8192, 8192), dict(cta_group=1, tileN=256, tileK=64, n_stage=4))]


def main():
    for (M, N, K), kw in CASES:
        def mk(i):
            A = (torch.rand(M, K, device="cuda") - 0.5).to(torch.bfloat16)
            B = (torch.rand(K, N, device="cuda") - 0.5).to(torch.bfloat16)
            return A, B, torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        rot = Rotating(mk, (M * K + K * N + M * N) * 2, max_sets=16)
        n = len(rot.sets)
        iters = max(n, 20 * n if M * N * K < 2 ** 33 else 2 * n)
        flops = 2.0 * M * N * K
        out = {"shape": [M, N, K], "sched": kw}
        ref = torch.matmul(rot.sets[0][0], rot.sets[0][1])
        for r in (0, 1, 2, 4, 6, 8, 12, 16, 1 << 20):
            s = alcop.make_schedule(raster=r, **kw)
            ms = time_graph(lambda i: alcop.matmul(rot.sets[i % n][0], rot.sets[i % n][1], s, out=rot.sets[i % n][2]),
                            iters=iters, reps_per_graph=n)
            ok = bool(torch.equal(rot.sets[0][2], ref))
            out[str(r if r < 1 << 20 else "mfast")] = round(flops / ms / 1e9, 1) if ok else "MISMATCH"
        ms = time_graph(lambda i: torch.matmul(rot.sets[i % n][0], rot.sets[i % n][1], out=rot.sets[i % n][2]),
                        iters=iters, reps_per_graph=n)
        out["cublas"] = round(flops / ms / 1e9, 1)
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
