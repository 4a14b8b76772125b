"""Library context (not a bench line): the pipelined GEMM with the model's
schedule beside torch.matmul (cuBLAS) on the same rotating inputs, both
captured in CUDA graphs.  Usage: python tools/cublas_compare.py [M N K ...]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2210_16691_b200 as alcop
from paper_2210_16691_b200.timing import Rotating, time_graph

SHAPES = [(4096, 768, 768), (4096, 3072, 768), (4096, 768, 3072), (4096, 4096, 4096), (8192, 8192, 8192),
          (16384, 4096, 4096)]


def run(M, N, K, extra=()):
    bytes_set = (M * K + K * N + M * N) * 2

    def mk(i):
        A = (torch.rand(M, K, device="cuda") - 0.5).to(torch.bfloat16)
        B = (torch.rand(K, N, device="cuda") - 0.5).to(torch.bfloat16)
        return A, B, torch.empty(M, N, device="cuda", dtype=torch.bfloat16)

    rot = Rotating(mk, bytes_set, max_sets=16)
    n = len(rot.sets)
    flops = 2.0 * M * N * K
    iters = max(n, 20 * n if M * N * K < 2 ** 33 else 2 * n)
    d = alcop.gemm_desc(M, N, K)
    res = {"shape": [M, N, K]}
    scheds = [("model", alcop.choose_schedule(d))] + list(extra)
    for name, s in scheds:
        ms = time_graph(lambda i: alcop.matmul(rot.sets[i % n][0], rot.sets[i % n][1], s, out=rot.sets[i % n][2]),
                        iters=iters, reps_per_graph=n)
        res[name] = {"tflops": round(flops / ms / 1e9, 1), "sched": repr(s)}
    ms = time_graph(lambda i: torch.matmul(rot.sets[i % n][0], rot.sets[i % n][1], out=rot.sets[i % n][2]),
                    iters=iters, reps_per_graph=n)
    res["cublas"] = round(flops / ms / 1e9, 1)
    A, B, C = rot.sets[0]
    alcop.matmul(A, B, scheds[0][1], out=C)
    ref = torch.matmul(A, B)
    res["max_rel_err_vs_cublas"] = float(((C.float() - ref.float()).abs().max() / ref.float().abs().max()).item())
    return res


def main():
    args = [int(x) for x in sys.argv[1:]]
    shapes = [tuple(args[i:i + 3]) for i in range(0, len(args), 3)] if args else SHAPES
    for M, N, K in shapes:
        print(json.dumps(run(M, N, K)), flush=True)


if __name__ == "__main__":
    main()
