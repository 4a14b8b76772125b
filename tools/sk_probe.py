"""Stream-K vs whole-tile CTA-pair GEMMs: CUDA-graph timing on rotating cold
inputs (> 2x L2), same schedule otherwise.   python tools/sk_probe.py"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2210_16691_b200 as alcop  # noqa: E402
from paper_2210_16691_b200.timing import Rotating, time_graph  # noqa: E402

SHAPES = [(4096, 3072, 768, 256, 6), (4096, 2304, 768, 256, 6), (4096, 4096, 4096, 256, 6),
          (4096, 3072, 768, 192, 6), (8192, 8192, 8192, 256, 6), (2048, 3072, 768, 256, 6),
          # 148 tiles = 2 full waves: stream-K splits nothing (pure scheduling overhead)
          (9472, 1024, 768, 256, 6), (9472, 1024, 3072, 256, 6),
          # long K, few waves: 80 tiles
          (2560, 2048, 16384, 256, 6),
          # the BERT N = 768 shapes: 64 pair tiles on 74 pairs (ffn2: 48 chunks per tile)
          (4096, 768, 3072, 192, 6), (4096, 768, 768, 192, 6)]
if os.environ.get("SK_SHAPES") == "bert":
    SHAPES = SHAPES[-2:]
if len(sys.argv) > 1:
    SHAPES = SHAPES[int(sys.argv[1]):]


def main():
    alcop.set_stream_k_workspace(256 << 20)  # caller-owned stream-K workspace
    res = {}
    for M, N, K, tn, st in SHAPES:
        rot = Rotating(lambda i: ((torch.rand((M, K), device="cuda") - 0.5).to(torch.bfloat16),
                                  (torch.rand((K, N), device="cuda") - 0.5).to(torch.bfloat16),
                                  torch.empty((M, N), device="cuda", dtype=torch.bfloat16)),
                       (M * K + K * N + M * N) * 2, max_sets=16)
        nr = len(rot.sets)
        row = {}
        for rep in range(2):
            for sk in (0, 1):
                s = alcop.make_schedule(tileN=tn, tileK=64, n_stage=st, cta_group=2, stream_k=sk)

                def run(i, s=s):
                    A, B, C = rot.sets[i % nr]
                    alcop.matmul(A, B, s, out=C)
                run(0)
                ms = time_graph(run, iters=max(8, 2 * nr), warmup=3, reps_per_graph=nr)
                tf = 2.0 * M * N * K / (ms * 1e-3) / 1e12
                row["sk%d" % sk] = max(row.get("sk%d" % sk, 0), round(tf, 1))
        res["%dx%dx%d/%d" % (M, N, K, tn)] = row
        print(M, N, K, tn, row, flush=True)
        del rot
        torch.cuda.empty_cache()
    print(json.dumps(res))


if __name__ == "__main__":
    main()
