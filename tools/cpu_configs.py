"""CPU columns of the per-config table (SURVEY §8d "Reference CPU path"):
for every BASELINE config, the reference interpreter's time on this host
(pipec::run on the transformed program, `oracle/_ref/ref_driver time`) and the
C oracle's (fp32-accumulate, OpenMP on all cores) — measured on a bounded
sample and extrapolated by the per-MMA cost (labelled), except C1 which runs
whole.  C4 (conv) has no reference CPU path: only the oracle's direct conv.

    python tools/cpu_configs.py [--out profiles/cpu_configs_r02.json] [--bench profiles/bench_r02.json]

Test/measurement infrastructure: executes oracle/ only as the baseline.
"""
import argparse
import json
import os
import platform
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import numpy as np  # noqa: E402
from oracle import coracle  # noqa: E402

CORES = os.cpu_count() or 1


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor()


def ref_blocks(blocks):
    """blocks: list of (m, n, K); all run concurrently; returns (makespan_s, mma count)."""
    drv = bench._ref_driver()
    tmp = tempfile.mkdtemp()
    ps = []
    t0 = time.perf_counter()
    for i, (m, n, K) in enumerate(blocks):
        sp = os.path.join(tmp, "b%d.txt" % i)
        with open(sp, "w") as f:
            f.write(bench._ref_sample_script(m, n, K))
        ps.append(subprocess.Popen([drv, "time", "--M", str(m), "--N", str(n), "--K", str(K), "--script", sp,
                                    "--mode", "stale", "--seed", str(i)], stdout=subprocess.PIPE,
                                   stderr=subprocess.PIPE, text=True))
    outs = [p.communicate() for p in ps]
    dt = time.perf_counter() - t0
    for p, (_, e) in zip(ps, outs):
        if p.returncode:
            raise RuntimeError(e)
    return dt, sum(m * n * K for m, n, K in blocks)


def ref_gemm(M, N, K, batch, rows):
    """Reference interpreter on CORES concurrent rows x min(N,128) blocks of
    one GEMM (full K); the job's time on this host is extrapolated from the
    measured MMA rate (the interpreter's cost is linear in m*n*K)."""
    n = min(N, 128)
    dt, mmas = ref_blocks([(rows, n, K)] * CORES)
    rate = mmas / dt  # MMA statements per second, all cores
    full = M * N * K * batch
    return {"sample": "%d concurrent %dx%dx%d blocks" % (CORES, rows, n, K), "sample_s": round(dt, 2),
            "ns_per_mma_per_core": round(dt * CORES / mmas * 1e9, 1),
            "est_s": round(full / rate, 1), "extrapolated": True}


def oracle_gemm(M, N, K, batch, rows):
    A = coracle.to_dtype(np.ones((rows, K), np.float32), "bf16")
    B = coracle.to_dtype(np.ones((K, N), np.float32), "bf16")
    coracle.gemm(A, B, "bf16", "bf16")
    t0 = time.perf_counter()
    coracle.gemm(A, B, "bf16", "bf16")
    dt = time.perf_counter() - t0
    frac = rows / M / batch
    return {"sample": "%d of %d rows%s" % (rows, M, " x 1 of %d batch" % batch if batch > 1 else ""),
            "sample_s": round(dt, 3), "est_s": round(dt / frac, 2), "extrapolated": frac < 1,
            "gflops": round(2.0 * rows * N * K / dt / 1e9, 1)}


def oracle_conv(H, C, K, R, st, pd, nimg):
    x = coracle.to_dtype(np.ones((nimg, H, H, C), np.float32), "bf16")
    w = coracle.to_dtype(np.ones((K, R, R, C), np.float32), "bf16")
    t0 = time.perf_counter()
    coracle.conv2d(x, w, (st, st), (pd, pd), "bf16", "bf16")
    return time.perf_counter() - t0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "cpu_configs_r02.json"))
    ap.add_argument("--bench", default=os.path.join(ROOT, "profiles", "bench_r02.json"))
    ap.add_argument("--ref-rows", type=int, default=64)
    args = ap.parse_args()
    coracle.build()
    gpu = {}
    if args.bench and os.path.exists(args.bench):
        with open(args.bench) as f:
            gpu = json.load(f)
    res = {"host": {"cores": CORES, "cpu": cpu_model()}, "configs": {}}
    cfg = res["configs"]

    # C1: the whole problem through the reference (16 output tiles, concurrent)
    dt, _ = ref_blocks([(128, 128, 512)] * 16)
    c1 = {"flops": 2.0 * 512 ** 3, "reference": {"sample": "whole C1: 16 concurrent 128x128x512 tile runs",
                                                 "est_s": round(dt, 2), "extrapolated": False},
          "oracle": oracle_gemm(512, 512, 512, 1, 512)}
    if "config1_512" in gpu:
        g = gpu["config1_512"]
        c1["gpu_us"] = min(g[k]["us"] for k in ("reference_schedule_wrap", "reference_schedule_fused", "model_pick"))
    cfg["C1_512_f16"] = c1

    # C2: BERT-base layer GEMMs (fused QKV form of the bench)
    for name, M, N, K in bench.BERT_GEMMS:
        e = {"flops": 2.0 * M * N * K, "reference": ref_gemm(M, N, K, 1, args.ref_rows),
             "oracle": oracle_gemm(M, N, K, 1, 256)}
        per_gemm = gpu.get("per_gemm") or gpu.get("bert_layer", {}).get("per_gemm", {})  # r01 / r02 line layout
        if name in per_gemm:
            e["gpu_us"] = round(per_gemm[name]["ms"] * 1e3, 2)
        cfg["C2_" + name] = e

    # C3: attention BMMs, batch*heads 192
    for name, (M, N, K) in (("qk_t", (512, 512, 64)), ("pv", (512, 64, 512))):
        e = {"flops": 2.0 * M * N * K * 192, "reference": ref_gemm(M, N, K, 192, args.ref_rows),
             "oracle": oracle_gemm(M, N, K, 192, 512)}
        g = gpu.get("bmm_attention", {}).get("gemms", {}).get(name)
        if g:
            e["gpu_us"] = round(e["flops"] / (g["tflops_aggregate"] * 1e12) * 1e6, 2)
        cfg["C3_" + name] = e

    # C4: ResNet-50 convs, batch 256: no reference CPU path; oracle direct conv on 2 images, x128
    tot = 0.0
    fl = 0.0
    for (name, H, C, K, R, st, pd, rep) in bench.RESNET50_CONVS:
        t = oracle_conv(H, C, K, R, st, pd, 2)
        P = (H + 2 * pd - R) // st + 1
        tot += t * 128 * rep
        fl += 2.0 * 256 * P * P * K * R * R * C * rep
    e = {"flops": fl, "reference": None, "reference_note": "no conv in the reference (SURVEY §8c)",
         "oracle": {"sample": "2 of 256 images per layer (direct conv)", "est_s": round(tot, 1),
                    "extrapolated": True}}
    g = gpu.get("resnet50_convs_b256")
    if g:
        e["gpu_us"] = round(fl / (g["tflops_aggregate"] * 1e12) * 1e6, 1)
    cfg["C4_resnet50_b256"] = e

    # C5: squares (reference extrapolated from a per-MMA rate at this K)
    for n in (4096, 8192, 12288, 16384):
        e = {"flops": 2.0 * n ** 3, "reference": ref_gemm(n, n, n, 1, args.ref_rows),
             "oracle": oracle_gemm(n, n, n, 1, max(8, 256 * 4096 // n))}
        g = gpu.get("large_square_m_sharded", {}).get("sizes", {}).get(str(n))
        if g:
            e["gpu_us"] = round(e["flops"] / (g["tflops_aggregate"] * 1e12) * 1e6, 1)
        elif str(n) in gpu.get("per_square", {}):  # r02 line: the headline squares, each timed alone
            e["gpu_us"] = round(gpu["per_square"][str(n)]["ms"] * 1e3, 1)
        cfg["C5_%d" % n] = e

    for e in cfg.values():
        if "gpu_us" in e:
            if e.get("reference"):
                e["gpu_speedup_vs_reference"] = round(e["reference"]["est_s"] / (e["gpu_us"] * 1e-6))
            e["gpu_speedup_vs_oracle"] = round(e["oracle"]["est_s"] / (e["gpu_us"] * 1e-6))
    with open(args.out, "w") as f:
        json.dump(res, f, indent=1)
    for k, e in cfg.items():
        r = e.get("reference") or {}
        print("%-20s ref %10s s%s  oracle %9s s  gpu %s us" % (k, r.get("est_s", "-"), "*" if r.get("extrapolated") else " ",
                                                              e["oracle"]["est_s"], e.get("gpu_us", "-")))


if __name__ == "__main__":
    main()
