"""Schedule grid for the BERT-layer shapes (incl. the fused QKV projection
4096x2304x768) with cuBLAS beside it (context only), CUDA-graph timing on
rotating inputs > 2x L2.  Usage: python tools/bert_probe.py [M N K ...]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2210_16691_b200 as alcop
from paper_2210_16691_b200.timing import Rotating, time_graph

SHAPES = [(4096, 768, 768), (4096, 2304, 768), (4096, 3072, 768), (4096, 768, 3072)]


def run(M, N, K, lay):
    bytes_set = (M * K + K * N + M * N) * 2

    def mk(i):
        A = (torch.rand(M, K, device="cuda") - 0.5).to(torch.bfloat16)
        B = (torch.rand(K, N, device="cuda") - 0.5).to(torch.bfloat16)
        if lay == alcop.B_NK:
            B = B.t().contiguous()
        return A, B, torch.empty(M, N, device="cuda", dtype=torch.bfloat16)

    rot = Rotating(mk, bytes_set, max_sets=16)
    n = len(rot.sets)
    flops = 2.0 * M * N * K
    iters = 20 * n
    d = alcop.gemm_desc(M, N, K, 1, alcop.BF16, alcop.BF16, lay)
    pick = alcop.choose_schedule(d)
    rows = []
    for cg in (1, 2):
        for tn in (64, 128, 192, 256):
            for tk in (64, 128):
                for st in range(2, 13):
                    s = alcop.make_schedule(tileN=tn, tileK=tk, n_stage=st, n_stage_inner=2, cta_group=cg)
                    try:
                        alcop.validate(d, s)
                    except alcop.AlcopError:
                        continue
                    ms = time_graph(lambda i, s=s: alcop.matmul(rot.sets[i % n][0], rot.sets[i % n][1], s,
                                                                out=rot.sets[i % n][2], b_layout=lay), iters=iters, reps_per_graph=n)
                    rows.append((round(flops / ms / 1e9, 1), cg, tn, tk, st, round(ms * 1e3, 2)))
    ms = time_graph(lambda i: alcop.matmul(rot.sets[i % n][0], rot.sets[i % n][1], pick, out=rot.sets[i % n][2],
                                                  b_layout=lay),
                    iters=iters, reps_per_graph=n)
    ms_cb = time_graph(lambda i: torch.matmul(rot.sets[i % n][0],
                                                  rot.sets[i % n][1].t() if lay == alcop.B_NK else rot.sets[i % n][1],
                                                  out=rot.sets[i % n][2]),
                       iters=iters, reps_per_graph=n)
    rows.sort(reverse=True)
    return {"shape": [M, N, K], "b_layout": "NK" if lay == alcop.B_NK else "KN", "pick": repr(pick), "pick_tflops": round(flops / ms / 1e9, 1),
            "cublas_tflops": round(flops / ms_cb / 1e9, 1), "top": rows[:12],
            "best_per_cg_tn": {"%d/%d" % (cg, tn): max([r for r in rows if r[1] == cg and r[2] == tn] or [None])
                               for cg in (1, 2) for tn in (64, 128, 192, 256)}}


def main():
    lay = alcop.B_NK if "--nk" in sys.argv else alcop.B_KN
    args = [int(x) for x in sys.argv[1:] if not x.startswith("--")]
    shapes = [tuple(args[i:i + 3]) for i in range(0, len(args), 3)] if args else SHAPES
    for M, N, K in shapes:
        print(json.dumps(run(M, N, K, lay)), flush=True)


if __name__ == "__main__":
    main()
