"""One BERT-layer step (the bench's fused-QKV decomposition) with the
bench's schedules, as plain launches for ncu (measurement tool):
    ncu ... -k regex:alcop python tools/profile_step.py --bench gpurun_out/bench.json --steps N
Launch order per step: qkv_proj, o_proj, ffn1, ffn2 (tools/ncu_summary.py
labels the captured launches in that order).  Inputs rotate over 3 sets."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2210_16691_b200 as alcop
from bench import BERT_GEMMS


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--bench", help="bench.py JSON line whose config.schedules to use (default: model picks)")
    ap.add_argument("--steps", type=int, default=4)
    args = ap.parse_args()
    scheds = {}
    if args.bench:
        with open(args.bench) as f:
            line = json.loads(f.read().strip().splitlines()[-1])
        scheds = {tuple(map(int, k.split("x"))): alcop.default_schedule(**v)
                  for k, v in line["config"]["schedules"].items()}
    sets = []
    for _ in range(3):
        one = []
        for name, M, N, K in BERT_GEMMS:
            A = (torch.rand(M, K, device="cuda") - 0.5).to(torch.bfloat16)
            B = (torch.rand(K, N, device="cuda") - 0.5).to(torch.bfloat16)
            C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
            s = scheds.get((M, N, K)) or alcop.choose_schedule(alcop.gemm_desc(M, N, K))
            one.append((A, B, C, s))
        sets.append(one)
    for i in range(args.steps):
        for A, B, C, s in sets[i % 3]:
            alcop.matmul(A, B, s, out=C)
    torch.cuda.synchronize()
    print("profile_step: %d steps x %d GEMMs" % (args.steps, len(BERT_GEMMS)),
          {n: repr(t[3]) for (n, *_), t in zip(BERT_GEMMS, sets[0])})


if __name__ == "__main__":
    main()
