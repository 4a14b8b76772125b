"""Host<->device copy bandwidth of this box (pinned memory): H2D alone, D2H
alone, and both directions at once on two streams.  Bounds the bench's e2e
number (the host-buffer entry point moves every step's A, B in and C out).

    python tools/pcie_probe.py [--mb 64] [--bench profiles/bench_r01.json]
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def timed(fn, iters=10):
    fn()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters * 1e-3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mb", type=int, default=64)
    ap.add_argument("--bench", default=None)
    args = ap.parse_args()
    n = args.mb << 20
    h_in = torch.empty(n, dtype=torch.uint8).pin_memory()
    h_out = torch.empty(n, dtype=torch.uint8).pin_memory()
    d_in = torch.empty(n, dtype=torch.uint8, device="cuda")
    d_out = torch.ones(n, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    cur = torch.cuda.current_stream()

    def both():
        s1.wait_stream(cur)
        s2.wait_stream(cur)
        with torch.cuda.stream(s1):
            d_in.copy_(h_in, non_blocking=True)
        with torch.cuda.stream(s2):
            h_out.copy_(d_out, non_blocking=True)
        cur.wait_stream(s1)
        cur.wait_stream(s2)

    t_h2d = timed(lambda: d_in.copy_(h_in, non_blocking=True))
    t_d2h = timed(lambda: h_out.copy_(d_out, non_blocking=True))
    t_both = timed(both)
    res = {"bytes": n, "h2d_gbs": round(n / t_h2d / 1e9, 1), "d2h_gbs": round(n / t_d2h / 1e9, 1),
           "bidirectional_gbs_each": round(n / t_both / 1e9, 1)}
    if args.bench and os.path.exists(args.bench):
        import bench
        with open(args.bench) as f:
            b = json.load(f)
        e = b["e2e"]
        flops = bench.step_flops()
        # lower bound on the e2e step: all copies at the measured rates, the two
        # directions fully overlapped, kernels hidden
        t_min = max(e["h2d_bytes_per_step"] / (res["bidirectional_gbs_each"] * 1e9),
                    e["d2h_bytes_per_step"] / (res["bidirectional_gbs_each"] * 1e9))
        t_ser = e["h2d_bytes_per_step"] / (res["h2d_gbs"] * 1e9) + e["d2h_bytes_per_step"] / (res["d2h_gbs"] * 1e9)
        res["e2e_bound_tflops_overlapped"] = round(flops / t_min / 1e12, 1)
        res["e2e_bound_tflops_serialized"] = round(flops / t_ser / 1e12, 1)
        res["e2e_measured_tflops"] = e["value"]
    print(json.dumps(res))


if __name__ == "__main__":
    main()
