"""Timeline of the bench's e2e step (alcop_gemm_host_async per GEMM of the
BERT layer, pinned host buffers) from a CUPTI trace (torch.profiler): busy time
of the H2D engine, the D2H engine and the kernels, their overlap, and the
idle gaps — what keeps the step above its PCIe bound (tools/pcie_probe.py).

    python tools/e2e_probe.py [--steps 5]
"""
import argparse
import ctypes
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2210_16691_b200 as alcop  # noqa: E402


def union(iv):
    iv = sorted(iv)
    out = []
    for a, b in iv:
        if out and a <= out[-1][1]:
            out[-1][1] = max(out[-1][1], b)
        else:
            out.append([a, b])
    return out


def total(iv):
    return sum(b - a for a, b in iv)


def inter(x, y):
    i = j = 0
    s = 0.0
    while i < len(x) and j < len(y):
        a = max(x[i][0], y[j][0])
        b = min(x[i][1], y[j][1])
        if b > a:
            s += b - a
        if x[i][1] < y[j][1]:
            i += 1
        else:
            j += 1
    return s


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--sync-each-step", type=int, default=1)
    args = ap.parse_args()
    lib = alcop.load_library()
    dev = torch.device("cuda", 0)
    gemms = bench.BERT_GEMMS
    descs, scheds, host, wss = [], [], [], []
    for _, M, N, K in gemms:
        d = alcop.gemm_desc(M, N, K, 1, alcop.BF16, alcop.BF16, alcop.B_KN)
        descs.append(d)
        scheds.append(alcop.choose_schedule(d))
        host.append(((torch.rand((M, K)) - 0.5).to(torch.bfloat16).pin_memory(),
                     (torch.rand((K, N)) - 0.5).to(torch.bfloat16).pin_memory(),
                     torch.empty((M, N), dtype=torch.bfloat16).pin_memory()))
        wss.append(torch.empty(lib.alcop_gemm_workspace_bytes(ctypes.byref(d)), dtype=torch.uint8, device=dev))
    sp = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)

    def step():
        for d, s, (A, B, C), ws in zip(descs, scheds, host, wss):
            rc = lib.alcop_gemm_host_async(ctypes.byref(d), ctypes.byref(s), ctypes.c_void_p(A.data_ptr()),
                                           ctypes.c_void_p(B.data_ptr()), ctypes.c_void_p(C.data_ptr()),
                                           ctypes.c_void_p(ws.data_ptr()), sp)
            assert rc == 0
        if args.sync_each_step:
            torch.cuda.synchronize()

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / args.steps
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(args.steps):
            step()
        torch.cuda.synchronize()
    h2d, d2h, ker = [], [], []
    for e in prof.events():
        if e.device_type != torch.autograd.DeviceType.CUDA:
            continue
        iv = (e.time_range.start, e.time_range.end)
        n = e.name.lower()
        if "htod" in n or "h2d" in n:
            h2d.append(iv)
        elif "dtoh" in n or "d2h" in n:
            d2h.append(iv)
        elif "alcop" in n:
            ker.append(iv)
    H, D, Kk = union(h2d), union(d2h), union(ker)
    allv = union(h2d + d2h + ker)
    span = allv[-1][1] - allv[0][0]
    res = {"wall_ms_per_step": round(wall * 1e3, 3), "trace_span_ms_per_step": round(span / args.steps / 1e3, 3),
           "h2d_busy_ms": round(total(H) / args.steps / 1e3, 3), "d2h_busy_ms": round(total(D) / args.steps / 1e3, 3),
           "kernel_busy_ms": round(total(Kk) / args.steps / 1e3, 3),
           "h2d_d2h_overlap_ms": round(inter(H, D) / args.steps / 1e3, 3),
           "idle_ms": round((span - total(allv)) / args.steps / 1e3, 3),
           "n_h2d": len(h2d), "n_d2h": len(d2h), "n_kernels": len(ker),
           "tflops_wall": round(bench.step_flops() / wall / 1e12, 1)}
    # one step's event list (relative us), first step
    first = sorted([(a, b, "H") for a, b in h2d] + [(a, b, "D") for a, b in d2h] + [(a, b, "K") for a, b in ker])
    base = first[0][0]
    per = len(first) // args.steps
    res["step0"] = [[k, round(a - base, 1), round(b - base, 1)] for a, b, k in first[:per]]
    print(json.dumps(res))


if __name__ == "__main__":
    main()
