"""Sustained throughput of the headline step (squares 4096..16384 once each,
one CUDA graph) per raster-group setting, and cuBLAS (torch.matmul) on the
same step, each run back to back for ~2 s of device time (the power-capped
regime the bench's timed region is in), three alternating rounds, median.
Measurement tool: python tools/sustained_probe.py [--seconds 2]"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2210_16691_b200 as alcop  # noqa: E402
from paper_2210_16691_b200 import workloads as W  # noqa: E402


def graph_of(fn):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    return g


def sustained(g, step_ms_guess, seconds, nv=None):
    import threading
    import time
    n = max(3, int(seconds * 1e3 / step_ms_guess))
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    samples, stop = [], threading.Event()

    def poll():
        while not stop.is_set():
            try:
                samples.append((nv[0].nvmlDeviceGetClockInfo(nv[1], nv[0].NVML_CLOCK_SM),
                                nv[0].nvmlDeviceGetPowerUsage(nv[1]) / 1e3))
            except Exception:
                pass
            time.sleep(0.01)
    t = threading.Thread(target=poll, daemon=True)
    if nv:
        t.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    stop.set()
    if nv:
        t.join()
    return e0.elapsed_time(e1) / n, samples


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=2.0)
    ap.add_argument("--rasters", default="0")
    a = ap.parse_args()
    ops = []
    for n in W.SQUARES:
        A = (torch.rand(n, n, device="cuda") - 0.5).to(torch.bfloat16)
        B = (torch.rand(n, n, device="cuda") - 0.5).to(torch.bfloat16)
        C = torch.empty(n, n, device="cuda", dtype=torch.bfloat16)
        ops.append((n, A, B, C, W.square_schedule(alcop, n, n)))
    flops = sum(2.0 * n ** 3 for n, *_ in ops)
    graphs = {}
    for r in [int(x) for x in a.rasters.split(",")]:
        def step(r=r):
            for n, A, B, C, s in ops:
                s2 = alcop.Schedule.from_buffer_copy(s)
                s2.raster = r
                alcop.matmul(A, B, s2, out=C)
        graphs["raster_%d" % r if r < 1 << 20 else "raster_mfast"] = graph_of(step)
    wide = alcop.make_schedule(tileN=512, tileK=64, n_stage=4, n_stage_inner=1, cta_group=2)
    for label, cut in (("wide_n>=8192", 8192), ("wide_all", 0)):
        def stepw(cut=cut):
            for n, A, B, C, s in ops:
                alcop.matmul(A, B, wide if n >= cut else s, out=C)
        graphs[label] = graph_of(stepw)
    graphs["cublas"] = graph_of(lambda: [torch.matmul(A, B, out=C) for n, A, B, C, s in ops])
    nv = None
    try:
        import pynvml
        pynvml.nvmlInit()
        nv = (pynvml, pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device()))
    except Exception:
        pass
    res = {k: [] for k in graphs}
    smp = {k: [] for k in graphs}
    for _ in range(3):
        for k, g in graphs.items():
            ms, sm = sustained(g, 9.0, a.seconds, nv)
            res[k].append(ms)
            smp[k] += sm[len(sm) // 4:]  # past the ramp
    out = {k: {"ms_per_step": round(statistics.median(v), 3),
               "tflops": round(flops / statistics.median(v) / 1e9, 1),
               "sm_mhz_median": statistics.median([c for c, _ in smp[k]]) if smp[k] else None,
               "power_w_median": round(statistics.median([p for _, p in smp[k]]), 1) if smp[k] else None}
           for k, v in res.items()}
    # each square alone, burst (short graph), current pick vs the wide tile
    from paper_2210_16691_b200.timing import time_graph
    alone = {}
    for n, A, B, C, s in ops:
        it = 20 if n <= 4096 else 4
        alone[str(n)] = {"pick_ms": round(time_graph(lambda i: alcop.matmul(A, B, s, out=C), iters=it), 4),
                         "wide_ms": round(time_graph(lambda i: alcop.matmul(A, B, wide, out=C), iters=it), 4),
                         "cublas_ms": round(time_graph(lambda i: torch.matmul(A, B, out=C), iters=it), 4)}
        ref = torch.matmul(A, B)
        alcop.matmul(A, B, wide, out=C)
        alone[str(n)]["wide_max_abs_diff_vs_cublas"] = float((C.float() - ref.float()).abs().max())
    print(json.dumps({"step": list(W.SQUARES), "seconds_per_measurement": a.seconds, "results": out,
                      "alone": alone}))


if __name__ == "__main__":
    main()
