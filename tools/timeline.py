"""Per-CTA globaltimer timeline of one pipelined-GEMM launch (debug tool).

python tools/timeline.py M N K tileN tileK stages [inner] [mode]
Stamps: 0 start, 1 setup done, 2 first TMA issued, 3 first full-wait passed,
4 last accumulator commit, 5 epilogue got first accumulator, 6 epilogue done,
7 CTA end.  Printed as microseconds after the earliest CTA start.
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2210_16691_b200 as alcop


def main():
    M, N, K, tN, tK, st = map(int, sys.argv[1:7])
    inner = int(sys.argv[7]) if len(sys.argv) > 7 else 2
    mode = int(sys.argv[8]) if len(sys.argv) > 8 else 1
    cg = int(sys.argv[9]) if len(sys.argv) > 9 else 1
    nctas = int(sys.argv[10]) if len(sys.argv) > 10 else 0
    batch = int(sys.argv[11]) if len(sys.argv) > 11 else 1
    shp = (batch,) if batch > 1 else ()
    lib = alcop.load_library()
    lib.alcop_debug_set_stamps.argtypes = [ctypes.c_void_p]
    A = torch.randn(shp + (M, K), device="cuda").to(torch.bfloat16)
    B = torch.randn(shp + (K, N), device="cuda").to(torch.bfloat16)
    C = torch.empty(shp + (M, N), device="cuda", dtype=torch.bfloat16)
    s = alcop.make_schedule(tileN=tN, tileK=tK, n_stage=st, n_stage_inner=inner, mode=mode, cta_group=cg,
                            num_ctas=nctas)
    stamps = torch.zeros(148 * 8 + 64 + 128 + 2, dtype=torch.int64, device="cuda")
    for _ in range(3):
        alcop.matmul(A, B, s, out=C)
    torch.cuda.synchronize()
    lib.alcop_debug_set_stamps(ctypes.c_void_p(stamps.data_ptr()))
    res = []
    mhz = []
    for rep in range(5):
        stamps.zero_()
        alcop.matmul(A, B, s, out=C)
        torch.cuda.synchronize()
        epi = stamps[148 * 8:148 * 8 + 64].view(16, 4).cpu().numpy().astype(np.int64)
        ch = stamps[148 * 8 + 64:148 * 8 + 192].view(2, 64).cpu().numpy().astype(np.int64)
        t = stamps[:148 * 8].view(148, 8).cpu().numpy().astype(np.int64)
        clk = stamps[148 * 8 + 192:148 * 8 + 194].cpu().numpy().astype(np.int64)
        mhz.append((clk[1] - clk[0]) / max(1, t[0, 7] - t[0, 0]) * 1e3)
        t = t[t[:, 0] > 0]
        t0 = t[:, 0].min()
        res.append((t - t0) / 1000.0)
    lib.alcop_debug_set_stamps(None)
    n = int((ch[1] > 0).sum())
    if n:
        base = ch[0, 0]
        print("CTA0 chunks (clk from first producer_acquire): acquire / consumer_wait passed")
        print("   acq ", [int(x - base) for x in ch[0, :n]])
        print("   wait", [int(x - base) for x in ch[1, :n]])
    nz = epi[epi[:, 0] > 0]
    if len(nz):
        base = nz[0, 0]
        print("epilogue CTA0 warp2 per chunk (clk from first chunk start): ldstart, ld+pack done, staging free, store issued")
        for row in nz:
            print("   ", [int(x - base) for x in row])
    print("CTA0 effective SM clock (clock64 / globaltimer): %s MHz" % [round(x) for x in mhz])
    names = ["start", "setup", "firstTMA", "firstFull", "lastCommit", "epiFirst", "epiDone", "end"]
    r = np.stack(res)  # reps x ctas x 8
    print("%s M=%d N=%d K=%d tile=128x%dx%d s=%d ctas=%d" % (s, M, N, K, tN, tK, st, r.shape[1]))
    for i, n in enumerate(names):
        col = r[:, :, i]
        print("  %-10s mean %7.2f  min %7.2f  max %7.2f us" % (n, col.mean(), col.min(), col.max()))


if __name__ == "__main__":
    main()
