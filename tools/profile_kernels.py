"""Launches one benchmarked kernel (or the headline step) a few times with the
bench's schedule, for ncu (measurement tool; numbers printed here are not
bench values).

    python tools/profile_kernels.py CASE [--reps N]

CASE: step (the headline step: squares 4096..16384 once each, repeated),
square4096 .. square16384, stem (ResNet-50 conv1, batch 256), l1_3x3
(56x56x64 -> 64, batch 256), l3_3x3, qkt / pv (attention BMMs, batch 192, the
tuned schedule), o_proj / ffn1 / ffn2 / qkv_proj (BERT GEMMs, tuned), chain
(the BERT layer as one alcop_gemm_chain launch).  Every launch writes a
fresh C buffer (rotating over copies > 2x L2 where C is small), so the
captured launch's DRAM writes are its own.
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2210_16691_b200 as alcop  # noqa: E402
from paper_2210_16691_b200 import workloads as W  # noqa: E402

L2 = 126 * 1024 * 1024


def rnd(*shape):
    return (torch.rand(shape, device="cuda") - 0.5).to(torch.bfloat16)


def gemm_case(M, N, K, batch=1, tune=False, sched=None):
    shp = (batch,) if batch > 1 else ()
    per = (M * K + K * N + M * N) * 2 * batch
    sets = [(rnd(*shp, M, K), rnd(*shp, K, N), torch.empty(shp + (M, N), device="cuda", dtype=torch.bfloat16))
            for _ in range(max(1, min(8, -(-2 * L2 // per))))]
    s = sched
    if s is None and M == N == K and batch == 1:
        s = W.square_schedule(alcop, M, N)
    if s is None:
        s = alcop.choose_schedule(alcop.gemm_desc(M, N, K, batch))
        if tune:
            s, _ = alcop.tune(*sets[0], budget=8)
    print("schedule", s, flush=True)
    i = {"k": 0}

    def run():
        A, B, C = sets[i["k"] % len(sets)]
        i["k"] += 1
        alcop.matmul(A, B, s, out=C)
    return run


def conv_case(name):
    L = [c for c in W.CONV_LAYERS if c.name == name][0]
    n = W.RESNET_BATCH
    hp = L.pad if L.halo else 0
    X = torch.zeros((n, L.H + 2 * hp, L.H + 2 * hp, L.Cs), device="cuda", dtype=torch.bfloat16)
    X[:, hp:hp + L.H, hp:hp + L.H, :L.C] = rnd(n, L.H, L.H, L.C)
    Wf = torch.zeros((L.K, L.R, L.R, L.Cs), device="cuda", dtype=torch.bfloat16)
    Wf[..., :L.C] = rnd(L.K, L.R, L.R, L.C)
    ys = [torch.empty((n, L.P, L.P, L.K), device="cuda", dtype=torch.bfloat16) for _ in range(2)]
    s = W.conv_schedule(alcop, L, n)
    print("schedule", s, flush=True)
    i = {"k": 0}

    def run():
        alcop.conv2d(X, Wf, (L.stride, L.stride), (L.pad, L.pad), sched=s, out=ys[i["k"] % 2], x_halo=L.halo)
        i["k"] += 1
    return run


def step_case():
    runs = [gemm_case(n, n, n) for n in W.SQUARES]

    def run():
        for r in runs:
            r()
    return run


def chain_case():
    sets = [[(rnd(M, K), rnd(K, N), torch.empty((M, N), device="cuda", dtype=torch.bfloat16))
             for _, M, N, K in W.BERT_GEMMS] for _ in range(4)]
    s = alcop.make_schedule(tileN=256, tileK=64, n_stage=6, cta_group=2)  # the bench's pick (CTA pairs)
    ws = torch.empty(1 << 16, dtype=torch.uint8, device="cuda")
    i = {"k": 0}

    def run():
        alcop.gemm_chain(sets[i["k"] % 4], s, workspace=ws)
        i["k"] += 1
    return run


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("case")
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    c = a.case
    if c == "step":
        run = step_case()
    elif c.startswith("square"):
        n = int(c[len("square"):])
        run = gemm_case(n, n, n)
    elif c == "stem":
        run = conv_case("conv1_7x7s2_3_64")
    elif c == "l1_3x3":
        run = conv_case("l1_3x3_64_64")
    elif c.startswith("conv_"):  # any ResNet-50 layer by name, e.g. conv_l3_1x1_256_1024
        run = conv_case(c[len("conv_"):])
    elif c == "l2_3x3":
        run = conv_case("l2_3x3_128")
    elif c == "l3_3x3":
        run = conv_case("l3_3x3_256")
    elif c in ("qkt", "pv"):
        M, N, K = (512, 512, 64) if c == "qkt" else (512, 64, 512)
        run = gemm_case(M, N, K, batch=W.BMM_BATCH, tune=True)
    elif c in [g[0] for g in W.BERT_GEMMS]:
        M, N, K = [g[1:] for g in W.BERT_GEMMS if g[0] == c][0]
        run = gemm_case(M, N, K, tune=True)
    elif c == "chain":
        run = chain_case()
    else:
        sys.exit("unknown case " + c)
    run()  # warm (module load, tensor-map encode) outside the profiled range
    torch.cuda.synchronize()
    torch.cuda.profiler.start()  # ncu --profile-from-start off captures from here
    for _ in range(a.reps):
        run()
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print("done", c)


if __name__ == "__main__":
    main()
