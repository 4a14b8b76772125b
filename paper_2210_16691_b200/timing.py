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
