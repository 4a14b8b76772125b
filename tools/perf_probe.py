"""Quick perf probe: TFLOP/s of the pipelined GEMM across shapes/schedules,
with torch.matmul (cuBLAS) beside it for context only."""
import itertools
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2210_16691_b200 as alcop
from paper_2210_16691_b200.timing import Rotating, time_fn


def probe(M, N, K, scheds, batch=1, iters=20):
    bytes_set = (M * K + K * N + M * N) * 2 * batch

    def mk(i):
        shp = (batch,) if batch > 1 else ()
        A = torch.randn(shp + (M, K), device="cuda").to(torch.bfloat16)
        B = torch.randn(shp + (K, N), device="cuda").to(torch.bfloat16)
        C = torch.empty(shp + (M, N), device="cuda", dtype=torch.bfloat16)
        return A, B, C

    rot = Rotating(mk, bytes_set, max_sets=8)
    flops = 2.0 * M * N * K * batch
    out = []
    for s in scheds:
        def f():
            A, B, C = rot.next()
            alcop.matmul(A, B, s, out=C)
        try:
            ms = time_fn(f, iters=iters)
        except Exception as e:  # noqa
            out.append((repr(s), "ERR " + str(e)))
            continue
        out.append((repr(s), round(flops / ms / 1e9, 1)))

    def g():
        A, B, C = rot.next()
        torch.matmul(A, B, out=C)
    ms = time_fn(g, iters=iters)
    out.append(("torch.matmul", round(flops / ms / 1e9, 1)))
    return out


def main():
    shapes = [(4096, 768, 768), (4096, 3072, 768), (4096, 768, 3072), (8192, 8192, 8192), (4096, 4096, 4096)]
    for (M, N, K) in shapes:
        scheds = []
        for tN, tK, st, mode in itertools.product([128, 256], [64, 128], [2, 3, 4, 6], [1, 0]):
            if (128 + tN) * tK * 2 * st > 225000:
                continue
            scheds.append(alcop.make_schedule(tileN=tN, tileK=tK, n_stage=st, n_stage_inner=2, mode=mode))
        scheds.append(alcop.make_schedule(tileN=256, tileK=64, n_stage=1, n_stage_inner=1))
        res = probe(M, N, K, scheds)
        res.sort(key=lambda r: -r[1] if isinstance(r[1], float) else 0)
        print(json.dumps({"shape": [M, N, K], "top": res[:8], "torch": [r for r in res if r[0] == "torch.matmul"],
                          "stage1": [r for r in res if "stages A/B=1/1" in r[0]]}), flush=True)


if __name__ == "__main__":
    main()
