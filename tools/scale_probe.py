"""Per-chunk time of the pipelined GEMM vs the number of persistent CTAs
(measurement tool): if the per-chunk time falls as CTAs are removed, the
main loop is bound by a chip-wide resource (L2 / HBM); if it stays, by a
per-SM one (TMA issue, ingress, MMA).  Cold (rotating > 2x L2) and warm
(one input set, L2-resident) operands.
Usage: python tools/scale_probe.py M N K tileN tileK stages cta_group [b_layout: kn|nk]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2210_16691_b200 as alcop
from paper_2210_16691_b200.timing import Rotating, time_graph


def main():
    M, N, K, tn, tk, st, cg = map(int, sys.argv[1:8])
    lay = alcop.B_NK if len(sys.argv) > 8 and sys.argv[8] == "nk" else alcop.B_KN

    def mk(i):
        A = (torch.rand(M, K, device="cuda") - 0.5).to(torch.bfloat16)
        B = (torch.rand(K, N, device="cuda") - 0.5).to(torch.bfloat16)
        if lay == alcop.B_NK:
            B = B.t().contiguous()
        return A, B, torch.empty(M, N, device="cuda", dtype=torch.bfloat16)

    rot = Rotating(mk, (M * K + K * N + M * N) * 2, max_sets=16)
    n = len(rot.sets)
    tiles = -(-M // (128 * cg)) * -(-N // tn)
    E = -(-K // tk)
    for ctas in (8, 16, 32, 64, 96, 128, 148):
        grid = min(ctas, tiles * cg)
        s = alcop.make_schedule(tileN=tn, tileK=tk, n_stage=st, n_stage_inner=2, cta_group=cg, num_ctas=grid)
        res = {"ctas": grid}
        for mode, nn in (("cold", n), ("warm", 1)):
            ms = time_graph(lambda i: alcop.matmul(rot.sets[i % nn][0], rot.sets[i % nn][1], s,
                                                   out=rot.sets[i % nn][2], b_layout=lay),
                            iters=max(8, 2 * nn), reps_per_graph=max(4, nn))
            per_cta_tiles = -(-tiles // (grid // cg))
            res[mode] = {"us": round(ms * 1e3, 2), "tflops": round(2.0 * M * N * K / ms / 1e9, 1),
                         "ns_per_chunk": round(ms * 1e6 / (per_cta_tiles * E), 1)}
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
