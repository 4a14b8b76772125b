"""§8(f) rank 4: the B200 two-level kernel simulation (alcop_simulate_kernel)
against device timings — t = 1 vs t = 2 TMEM accumulators (the inner level)
and FUSED vs WRAP (outer ring run-ahead vs per-tile restart) on shapes with
many tiles per CTA.  Prints one JSON line per case; --json PATH saves all."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2210_16691_b200 as alcop
from paper_2210_16691_b200.timing import Rotating, time_graph

SHAPES = [(8192, 8192, 256), (8192, 8192, 512), (8192, 4096, 1024), (4096, 4096, 2048)]
SCHEDS = [dict(tileN=256, tileK=64, n_stage=st, n_stage_inner=t, mode=m)
          for st in (1, 2, 4) for t in (1, 2) for m in (alcop.MODE_FUSED, alcop.MODE_WRAP)
          if not (m == alcop.MODE_WRAP and st == 1)]


def measure(M, N, K, scheds):
    def mk(i):
        A = (torch.rand(M, K, device="cuda") - 0.5).to(torch.bfloat16)
        B = (torch.rand(K, N, device="cuda") - 0.5).to(torch.bfloat16)
        return A, B, torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    rot = Rotating(mk, (M * K + K * N + M * N) * 2, max_sets=8)
    n = len(rot.sets)
    d = alcop.gemm_desc(M, N, K)
    rows = []
    for kw in scheds:
        s = alcop.make_schedule(**kw)
        ms = time_graph(lambda i: alcop.matmul(rot.sets[i % n][0], rot.sets[i % n][1], s, out=rot.sets[i % n][2]),
                        iters=10 * n, reps_per_graph=n)
        sim = alcop.simulate_kernel(d, s)
        rows.append({"shape": [M, N, K], **kw, "ms": ms, "sim_ms": sim["seconds"] * 1e3,
                     "pred_ms": alcop.predict(d, s)["seconds"] * 1e3})
    return rows


def main():
    out = sys.argv[sys.argv.index("--json") + 1] if "--json" in sys.argv else None
    allrows = []
    for M, N, K in SHAPES:
        rows = measure(M, N, K, SCHEDS)
        allrows += rows
        for r in rows:
            print(json.dumps(r), flush=True)
    if out:
        with open(out, "w") as f:
            json.dump(allrows, f)


if __name__ == "__main__":
    main()
