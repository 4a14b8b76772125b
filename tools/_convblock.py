"""Run bench.conv_block alone (debug of the conv block's per-layer numbers)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2210_16691_b200 as alcop
dev = torch.device("cuda", 0)
peaks = bench.load_peaks()
def attainable(fl, byts):
    return min(peaks["bf16_tflops"], fl / byts * peaks["hbm_gbs"] * 1e-3)
class A: pass
parity = {}
r = bench.conv_block(A(), torch, alcop, dev, 0, 1, bench.Ranks(0, 1, dev), parity, attainable)
print(r["tflops_aggregate"])
for l in r["layers"]:
    print(l["layer"], l["tflops"], l["model_pick_over_best_swept"], l["schedule"], l["best_swept"])
