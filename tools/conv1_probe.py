"""ResNet-50 conv1 (7x7/2, 3 -> 64, batch 256) paths, per schedule: the stem
kernel on NHWC4 (csrc/stem_sm100.cu, pixel-pair descriptors), the
one-box-per-filter-row kernel on the halo-padded NHWC8 input, and the
8-channel im2col path; all three outputs compared bit for bit."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2210_16691_b200 as alcop
from paper_2210_16691_b200.timing import time_graph


def main():
    n, H, C, Cs, K, R, st, pd = int(sys.argv[1]) if len(sys.argv) > 1 else 256, 224, 3, 8, 64, 7, 2, 3
    P = Q = (H + 2 * pd - R) // st + 1
    flops = 2.0 * n * P * Q * K * R * R * C
    Xh = torch.zeros((n, H + 2 * pd, H + 2 * pd, Cs), device="cuda", dtype=torch.bfloat16)
    Xh[:, pd:pd + H, pd:pd + H, :C] = (torch.rand((n, H, H, C), device="cuda") - 0.5).to(torch.bfloat16)
    X = Xh[:, pd:pd + H, pd:pd + H, :].contiguous()
    Wf = torch.zeros((K, R, R, Cs), device="cuda", dtype=torch.bfloat16)
    Wf[..., :C] = (torch.rand((K, R, R, C), device="cuda") - 0.5).to(torch.bfloat16)
    Y = torch.empty((n, P, Q, K), device="cuda", dtype=torch.bfloat16)
    Y2 = torch.empty_like(Y)
    out = {"bytes_min": Xh.numel() * 2 + Y.numel() * 2}
    for halo in (True, False):
        for tn, stg in ((64, 2), (64, 4), (64, 6), (64, 8), (64, 1)):
            s = alcop.make_schedule(tileN=tn, tileK=64, n_stage=stg, n_stage_inner=2 if stg > 1 else 1)
            src = Xh if halo else X
            ms = time_graph(lambda i: alcop.conv2d(src, Wf, (st, st), (pd, pd), sched=s, out=Y, x_halo=halo),
                            iters=6, warmup=2)
            out["%s_s%d" % ("stem" if halo else "im2col8", stg)] = {"ms": round(ms, 4), "tflops": round(flops / ms / 1e9, 1),
                                                                    "GBps": round(out["bytes_min"] / ms / 1e6, 1)}
    X4 = X[..., :4].contiguous()
    W4 = Wf[..., :4].contiguous()
    out["bytes_min_nhwc4"] = X4.numel() * 2 + Y.numel() * 2
    d = alcop.conv_desc(n, H, H, 4, K, R, R, (st, st), (pd, pd), alcop.BF16, alcop.BF16)
    pick = alcop.choose_conv_schedule(d)
    out["pairs_model_pick"] = pick.as_dict()
    for stg, inn in ((6, 2), (6, 1), (5, 1), (4, 2), (4, 1), (3, 1), (2, 2), (1, 1)):
        s = alcop.make_schedule(tileN=K, tileK=64, n_stage=stg, n_stage_inner=inn)
        try:
            ms = time_graph(lambda i: alcop.conv2d(X4, W4, (st, st), (pd, pd), sched=s, out=Y, x_halo=False),
                            iters=10, warmup=3)
        except alcop.AlcopError as e:
            out["pairs_s%d_a%d" % (stg, inn)] = str(e)[:40]
            continue
        out["pairs_s%d_a%d" % (stg, inn)] = {"ms": round(ms, 4), "tflops": round(flops / ms / 1e9, 1),
                                             "GBps": round(out["bytes_min_nhwc4"] / ms / 1e6, 1)}
    Y3 = torch.empty_like(Y)
    alcop.conv2d(Xh, Wf, (st, st), (pd, pd), out=Y, x_halo=True)
    alcop.conv2d(X, Wf, (st, st), (pd, pd), out=Y2)
    alcop.conv2d(X4, W4, (st, st), (pd, pd), out=Y3)
    out["stem_equals_im2col"] = bool(torch.equal(Y, Y2))
    out["pairs_equals_im2col"] = bool(torch.equal(Y3, Y2))
    print(json.dumps(out))


if __name__ == "__main__":
    main()
