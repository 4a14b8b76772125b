import sys, json, ctypes
sys.path.insert(0, '/root/repo')
import torch
import paper_2210_16691_b200 as alcop
from paper_2210_16691_b200.timing import Rotating, time_graph
lib = alcop.load_library()
M, N, K, nb = 512, 512, 64, 192
db = alcop.gemm_desc(M, N, K, nb, alcop.BF16, alcop.BF16, alcop.B_KN)
sb = alcop.choose_schedule(db)
rot = Rotating(lambda i: ((torch.rand((nb, M, K), device="cuda") - 0.5).to(torch.bfloat16), (torch.rand((nb, K, N), device="cuda") - 0.5).to(torch.bfloat16), torch.empty((nb, M, N), device="cuda", dtype=torch.bfloat16)), (M*K+K*N+M*N)*2*nb, max_sets=16)
nr = len(rot.sets)
def runb(i):
    A, B, C = rot.sets[i % nr]
    rc = lib.alcop_gemm(ctypes.byref(db), ctypes.byref(sb), ctypes.c_void_p(A.data_ptr()), ctypes.c_void_p(B.data_ptr()), ctypes.c_void_p(C.data_ptr()), ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    assert rc == 0
def runm(i):
    A, B, C = rot.sets[i % nr]
    alcop.matmul(A, B, sb, out=C)
byts = (M*K+K*N+M*N)*2*nb
out = {"nr": nr, "sched": repr(sb)}
for name, f in (("ctypes", runb), ("matmul", runm), ("ctypes2", runb)):
    ms = time_graph(f, iters=12*nr, warmup=3, reps_per_graph=nr)
    out[name] = round(byts / ms / 1e6, 1)
print(json.dumps(out))
