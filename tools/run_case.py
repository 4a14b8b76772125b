"""Runs one pipelined-GEMM configuration `--reps` times (for ncu captures).

python tools/run_case.py M N K tileN tileK stages [inner] [mode] [--reps R] [--batch B] [--layout kn|nk]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2210_16691_b200 as alcop


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("M", type=int)
    ap.add_argument("N", type=int)
    ap.add_argument("K", type=int)
    ap.add_argument("tileN", type=int)
    ap.add_argument("tileK", type=int)
    ap.add_argument("stages", type=int)
    ap.add_argument("inner", type=int, nargs="?", default=2)
    ap.add_argument("mode", type=int, nargs="?", default=1)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--layout", default="kn")
    a = ap.parse_args()
    shp = (a.batch,) if a.batch > 1 else ()
    A = torch.randn(shp + (a.M, a.K), device="cuda").to(torch.bfloat16)
    B = torch.randn(shp + ((a.K, a.N) if a.layout == "kn" else (a.N, a.K)), device="cuda").to(torch.bfloat16)
    C = torch.empty(shp + (a.M, a.N), device="cuda", dtype=torch.bfloat16)
    s = alcop.make_schedule(tileN=a.tileN, tileK=a.tileK, n_stage=a.stages, n_stage_inner=a.inner, mode=a.mode)
    lay = alcop.B_KN if a.layout == "kn" else alcop.B_NK
    for _ in range(a.reps):
        alcop.matmul(A, B, s, out=C, b_layout=lay)
    torch.cuda.synchronize()
    print("ok", s)


if __name__ == "__main__":
    main()
