"""Which base-offset makes a row-shifted 128B-swizzled descriptor read the
intended rows?  (semantics probe; tools/desc_probe.cu)"""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

lib = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "_bin", "libdesc_probe.so"))
g = torch.Generator().manual_seed(1)
A = torch.randint(-8, 8, (144, 64), generator=g).to(torch.bfloat16)
B = torch.randint(-8, 8, (64, 64), generator=g).to(torch.bfloat16)
Ad, Bd = A.cuda(), B.cuda()
out = {}
for shift in range(0, 10):
    row = {}
    for bo in range(8):
        D = torch.zeros(128, 64, device="cuda")
        rc = lib.desc_probe(ctypes.c_void_p(Ad.data_ptr()), ctypes.c_void_p(Bd.data_ptr()), ctypes.c_void_p(D.data_ptr()),
                            shift, bo)
        ref = A[shift:shift + 128].float() @ B.float().t()
        row[bo] = "ok" if rc == 0 and torch.equal(D.cpu(), ref) else ("rc%d" % rc if rc else "bad")
    out[shift] = row
print(json.dumps(out))
