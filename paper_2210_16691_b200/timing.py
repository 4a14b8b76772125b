"""Device timing helpers shared by bench.py and the schedule sweep.

CUDA events on the launching stream, warm-up first, synchronize on both
sides; L2 is defeated by rotating over input copies whose total footprint
exceeds 2x the 126 MB L2 (or by an explicit flush buffer).
"""
from __future__ import annotations

import torch

L2_BYTES = 126 * 1024 * 1024


class Rotating:
    """n copies of a GEMM's (A, B, C) so consecutive launches miss in L2."""

    def __init__(self, make_inputs, bytes_per_set, min_sets=2, max_sets=64):
        n = max(min_sets, min(max_sets, (2 * L2_BYTES + bytes_per_set - 1) // max(1, bytes_per_set)))
        self.sets = [make_inputs(i) for i in range(n)]
        self.i = 0

    def next(self):
        s = self.sets[self.i]
        self.i = (self.i + 1) % len(self.sets)
        return s


def time_fn(fn, iters=20, warmup=5, stream=None):
    """Mean device ms per call of fn() (fn launches on `stream`)."""
    stream = stream or torch.cuda.current_stream()
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    start = torch.cuda.Event(enable_timing=True)
    end = torch.cuda.Event(enable_timing=True)
    start.record(stream)
    for _ in range(iters):
        fn()
    end.record(stream)
    torch.cuda.synchronize()
    return start.elapsed_time(end) / iters


def time_graph(launch, iters=20, warmup=3, reps_per_graph=None):
    """Mean device ms per launch() call, with the launches captured into a
    CUDA graph so host launch overhead does not leak into short kernels.
    launch(i) enqueues one unit of work on the current stream (i = index of
    the call inside the graph, for rotating inputs)."""
    import os
    if os.environ.get("ALCOP_BENCH_GRAPHS", "1") == "0":  # profiling: plain launches
        cnt = {"i": 0}

        def f():
            launch(cnt["i"])
            cnt["i"] += 1
        return time_fn(f, iters=iters, warmup=warmup)
    reps = reps_per_graph or iters
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for i in range(warmup):
            launch(i)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(reps):
            launch(i)
    g.replay()
    torch.cuda.synchronize()
    start = torch.cuda.Event(enable_timing=True)
    end = torch.cuda.Event(enable_timing=True)
    n = max(1, iters // reps)
    start.record()
    for _ in range(n):
        g.replay()
    end.record()
    torch.cuda.synchronize()
    return start.elapsed_time(end) / (n * reps)
