"""CTA 0's MMA-thread timeline of one CTA-pair GEMM launch from the
-DGEMM_TRACE build (ALCOP_LIB=paper_2210_16691_b200/libalcop_gtrace.so):
per chunk, clock64 after the full-barrier wait and after the chunk's MMAs +
commit were issued, plus per tile the start and the
accumulator-free time; for one CTA per tile (cta_group 1) the producer's
acquire / issue clocks and the MMA warp's full-wait clocks per chunk.
Measurement only; --parse / --parse-single FILE summarise a saved run.
python tools/gemm_trace.py M N K tileN tileK stages [cta_group [inner]]"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2210_16691_b200 as alcop


def parse(path):
    """Per tile: clk from tile start to accumulator free, the chunks' full-wait
    times and the issue spans, relative to the first record."""
    recs = [int(l.split()[2]) for l in open(path) if l.startswith("T ")]
    base = None
    tiles = []
    for r in recs:
        v = r & ((1 << 61) - 1)
        base = v if base is None else base
        if r >> 62 & 1:
            tiles.append({"start": v - base, "acc_free": None, "chunks": []})
        elif r >> 61 & 1:
            tiles[-1]["acc_free"] = v - base
        else:
            tiles[-1]["chunks"].append(v - base)
    for t in tiles:
        w = t["chunks"][0::2]
        print("tile start %6d  acc free +%5d  chunk waits %s" % (
            t["start"], (t["acc_free"] or 0) - t["start"], [x - t["start"] for x in w]))


def parse_single(path):
    """Single-CTA kernel (P / C lines of the last launch in the file): per chunk
    the producer's acquire and issue-done clocks and the MMA warp's full-wait
    clock, relative to the first acquire."""
    runs, cur = [], None
    for line in open(path):
        if line.startswith("RUN"):
            cur = {"P": [], "C": []}
            runs.append(cur)
        elif cur is not None and line[:2] in ("P ", "C "):
            cur[line[0]].append(int(line.split()[2]))
    r = runs[-1]
    acq = [v for v in r["P"] if not v >> 62 & 1]
    iss = [v & ((1 << 62) - 1) for v in r["P"] if v >> 62 & 1]
    base = acq[0]
    print("acquire ", [v - base for v in acq])
    print("issued  ", [v - base for v in iss])
    print("issue   ", [b - a for a, b in zip(acq, iss)])
    print("full ok ", [v - base for v in r["C"]])


if sys.argv[1] == "--parse":
    parse(sys.argv[2])
    sys.exit(0)
if sys.argv[1] == "--parse-single":
    parse_single(sys.argv[2])
    sys.exit(0)
M, N, K, tn, tk, st = map(int, sys.argv[1:7])
cg = int(sys.argv[7]) if len(sys.argv) > 7 else 2
inner = int(sys.argv[8]) if len(sys.argv) > 8 else 2
A = (torch.rand(M, K, device="cuda") - 0.5).to(torch.bfloat16)
B = (torch.rand(K, N, device="cuda") - 0.5).to(torch.bfloat16)
C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
s = alcop.make_schedule(tileN=tn, tileK=tk, n_stage=st, cta_group=cg, n_stage_inner=inner)
for _ in range(3):  # the last launch is the warm one
    print("RUN", flush=True)
    alcop.matmul(A, B, s, out=C)
    torch.cuda.synchronize()
