"""Per-k-block clock64 timeline of CTA 0 (debug): producer acquire waits and
MMA-thread waits, to find the per-k-block critical path."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2210_16691_b200 as alcop
M, N, K, tN, tK, st = map(int, sys.argv[1:7])
lay = alcop.B_NK if len(sys.argv) > 7 and sys.argv[7] == "nk" else alcop.B_KN
lib = alcop.load_library()
lib.alcop_debug_set_stamps.argtypes = [ctypes.c_void_p]
A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
B = torch.randn(K, N, device="cuda").to(torch.bfloat16)
if lay == alcop.B_NK:
    B = B.t().contiguous()
C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
s = alcop.make_schedule(tileN=tN, tileK=tK, n_stage=st)
buf = torch.zeros(148 * 8 + 3 * 512 * 4, dtype=torch.int64, device="cuda")
for _ in range(2):
    alcop.matmul(A, B, s, out=C, b_layout=lay)
lib.alcop_debug_set_stamps(ctypes.c_void_p(buf.data_ptr()))
alcop.matmul(A, B, s, out=C, b_layout=lay)
torch.cuda.synchronize()
lib.alcop_debug_set_stamps(None)
kb = buf[148 * 8:].view(3, 512, 4).cpu().numpy()
t0 = kb[2, 1, 0]
n = min(512, K // tK * 2)
print(s, "per-kblock (cycles rel. to MMA wait #1)")
print(" kb | prodA wait-> ok expect tma | prodB wait->ok | mma waitA start  A ok  B ok")
for i in range(1, min(n, 60)):
    pa, pb, mm = kb[0, i], kb[1, i], kb[2, i]
    print("%3d | %8d %6d %6d %6d | %8d %6d | %8d %6d %6d" % (i, pa[0] - t0, pa[1] - pa[0], pa[2] - pa[1], pa[3] - pa[2],
                                                       pb[0] - t0, pb[1] - pb[0], mm[0] - t0, mm[1] - mm[0], mm[2] - mm[1]))
d = np.diff(kb[2, 1:n, 0])
print("mean cycles between MMA k-blocks:", d[len(d)//2:].mean())
