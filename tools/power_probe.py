"""Power-capped regime data for the B200 model's energy term (measurement tool).

For each square n and schedule: the sustained time per launch (the GEMM
back to back for --seconds of device time, after a warm-up, like the bench's
timed step), the exact L2 -> SM TMA bytes of the schedule, and (with
--mode ncu, under `ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum
--profile-from-start off`) one launch of each for its DRAM traffic.

    python tools/power_probe.py --mode time > gpurun_out/power_time.json
    ncu ... python tools/power_probe.py --mode ncu
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2210_16691_b200 as alcop  # noqa: E402

SIZES = (8192, 12288, 16384)
SCHEDS = {
    "pair256_s6": dict(tileN=256, tileK=64, n_stage=6, cta_group=2),
    "pair256_s6_r4": dict(tileN=256, tileK=64, n_stage=6, cta_group=2, raster=4),
    "pair192_s7": dict(tileN=192, tileK=64, n_stage=7, cta_group=2),
    "pair512_s4": dict(tileN=512, tileK=64, n_stage=4, n_stage_inner=1, cta_group=2),
    "pair512_s4_r4": dict(tileN=512, tileK=64, n_stage=4, n_stage_inner=1, cta_group=2, raster=4),
    "single256_s4": dict(tileN=256, tileK=64, n_stage=4, cta_group=1),
    "single128_s6": dict(tileN=128, tileK=64, n_stage=6, cta_group=1),
}


def l2_to_sm_bytes(n, s):
    """Exact TMA bytes: every tile loads its A rows and B columns for every chunk."""
    tm, tn, tk = s.tileM, s.tileN, s.tileK
    tiles = (-(-n // tm)) * (-(-n // tn))
    chunks = -(-n // tk)
    return tiles * chunks * (tm + tn) * tk * 2


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mode", default="time", choices=["time", "ncu"])
    ap.add_argument("--seconds", type=float, default=1.5)
    ap.add_argument("--sizes", default=",".join(map(str, SIZES)))
    ap.add_argument("--scheds", default="", help="name=tileN:tileK:stages:cta_group:inner:raster,... (default: SCHEDS)")
    a = ap.parse_args()
    scheds = SCHEDS
    if a.scheds:
        scheds = {}
        for item in a.scheds.split(","):
            name, spec = item.split("=")
            tn, tk, st, cg, inner, r = map(int, spec.split(":"))
            scheds[name] = dict(tileN=tn, tileK=tk, n_stage=st, cta_group=cg, n_stage_inner=inner, raster=r)
    res = []
    for n in map(int, a.sizes.split(",")):
        A = (torch.rand(n, n, device="cuda") - 0.5).to(torch.bfloat16)
        B = (torch.rand(n, n, device="cuda") - 0.5).to(torch.bfloat16)
        C = torch.empty(n, n, device="cuda", dtype=torch.bfloat16)
        for name, kw in scheds.items():
            s = alcop.make_schedule(**kw)
            alcop.matmul(A, B, s, out=C)
            torch.cuda.synchronize()
            if a.mode == "ncu":
                torch.cuda.profiler.start()
                alcop.matmul(A, B, s, out=C)
                torch.cuda.synchronize()
                torch.cuda.profiler.stop()
                print(json.dumps({"n": n, "sched": name}), flush=True)
                continue
            # warm the power state, then time a sustained run
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            alcop.matmul(A, B, s, out=C)
            e1.record()
            torch.cuda.synchronize()
            one = e0.elapsed_time(e1)
            reps = max(3, int(a.seconds * 1e3 / one))
            for _ in range(max(2, reps // 4)):
                alcop.matmul(A, B, s, out=C)
            e0.record()
            for _ in range(reps):
                alcop.matmul(A, B, s, out=C)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / reps
            res.append({"n": n, "sched": name, "schedule": s.as_dict(), "ms_sustained": round(ms, 4),
                        "tflops": round(2.0 * n ** 3 / ms / 1e9, 1), "flops": 2.0 * n ** 3,
                        "l2_to_sm_B": l2_to_sm_bytes(n, s)})
            print(json.dumps(res[-1]), flush=True)
        del A, B, C
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
