"""Summarise the per-kernel `ncu --set full` captures of tools/ncu_round.sh
(gpurun_out/ncu_<case>_raw.csv) and the headline step's launch list
(gpurun_out/launches_step.csv) into profiles/ (measurement tool).

    python tools/ncu_kernels_summary.py [--round r02]

Per kernel: duration, SM clock, tensor-pipe activity, DRAM read / write bytes
(+ the bytes written into L2, which is where a C smaller than L2 sits when the
kernel ends), L2 -> SM (TMA) bytes, and the algorithmic FLOPs / compulsory
bytes of the case, so traffic / compulsory shows re-reads."""
import argparse
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2210_16691_b200 import workloads as W  # noqa: E402

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "sector": 32, "ns": 1e-3, "nsecond": 1e-3,
         "us": 1, "usecond": 1, "ms": 1e3, "msecond": 1e3, "%": 1, "Ghz": 1e3, "Mhz": 1, "hz": 1e-6, "cycle": 1}
WANT = {
    "duration_us": "gpu__time_duration.sum",
    "sm_mhz": "sm__cycles_elapsed.avg.per_second",
    "tensor_pipe_active_pct": "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "tensor_pipe_active_realtime_pct": "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "dram_read_B": "dram__bytes_read.sum",
    "dram_write_B": "dram__bytes_write.sum",
    "l2_write_B": "lts__t_sectors_op_write.sum",
    "l2_to_sm_tma_B": "l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld.sum",
    "dram_throughput_pct": "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm_throughput_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "registers_per_thread": "launch__registers_per_thread",
}


def case_work(case):
    """(FLOPs, compulsory bytes, description) of a profile_kernels.py case."""
    if case.startswith("square"):
        n = int(case[6:])
        return 2.0 * n ** 3, 2 * 3 * n * n, "square %d^3 bf16" % n
    if case in ("qkt", "pv"):
        M, N, K = (512, 512, 64) if case == "qkt" else (512, 64, 512)
        b = W.BMM_BATCH
        return 2.0 * M * N * K * b, 2 * b * (M * K + K * N + M * N), "attention %s batch %d" % (case, b)
    if case.startswith("conv_"):
        L = [c for c in W.CONV_LAYERS if c.name == case[len("conv_"):]][0]
        return L.flops(W.RESNET_BATCH), L.compulsory_bytes(W.RESNET_BATCH), "ResNet-50 %s batch 256" % L.name
    convs = {"stem": "conv1_7x7s2_3_64", "l1_3x3": "l1_3x3_64_64", "l2_3x3": "l2_3x3_128", "l3_3x3": "l3_3x3_256"}
    if case in convs:
        L = [c for c in W.CONV_LAYERS if c.name == convs[case]][0]
        return L.flops(W.RESNET_BATCH), L.compulsory_bytes(W.RESNET_BATCH), "ResNet-50 %s batch 256" % L.name
    bert = {g[0]: g[1:] for g in W.BERT_GEMMS}
    if case in bert:
        M, N, K = bert[case]
        return 2.0 * M * N * K, 2 * (M * K + K * N + M * N), "BERT %s %dx%dx%d" % (case, M, N, K)
    if case == "chain":
        f = sum(2.0 * M * N * K for _, M, N, K in W.BERT_GEMMS)
        b = sum(2 * (M * K + K * N + M * N) for _, M, N, K in W.BERT_GEMMS)
        return f, b, "BERT layer, 4 GEMMs in one alcop_gemm_chain launch"
    return None, None, case


def read_raw(path):
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", ""),
             "grid": r[hdr.index("Grid Size")], "block": r[hdr.index("Block Size")]}
        for key, metric in WANT.items():
            if metric in hdr:
                i = hdr.index(metric)
                try:
                    d[key] = float(r[i].replace(",", "")) * SCALE.get(units[i], 1)
                except ValueError:
                    pass
        out.append(d)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--round", default="r02")
    ap.add_argument("--src", default=os.path.join(ROOT, "gpurun_out"))
    a = ap.parse_args()
    kernels = {}
    for f in sorted(os.listdir(a.src)):
        if not (f.startswith("ncu_") and f.endswith("_raw.csv")):
            continue
        case = f[4:-8]
        rows = read_raw(os.path.join(a.src, f))
        if not rows:
            continue
        d = rows[0]
        fl, cb, what = case_work(case)
        d["case"] = what
        if fl:
            d["algorithmic_flops"] = fl
            d["compulsory_B"] = cb
            d["tflops_under_ncu"] = round(fl / (d["duration_us"] * 1e-6) / 1e12, 1)
            d["dram_read_over_compulsory_inputs"] = round(d.get("dram_read_B", 0) / max(1, cb), 2)
        kernels[case] = {k: (round(v, 3) if isinstance(v, float) else v) for k, v in d.items()}
    out = {"source": "ncu --set full --import-source on --clock-control none, one launch per case "
                     "(tools/ncu_round.sh -> tools/profile_kernels.py CASE; the bench's schedules). Serialized, "
                     "cache-flushed replay: compare shares and traffic, not absolute times. dram_write_B counts only "
                     "write-backs inside the launch: a C smaller than L2 is still dirty in L2 when the kernel ends "
                     "(l2_write_B is what the kernel wrote into L2).",
           "kernels": kernels}
    dst = os.path.join(ROOT, "profiles", "ncu_kernels_%s.json" % a.round)
    if os.path.exists(dst):  # keep the cases not recaptured this time (marked as from an earlier capture)
        old = json.load(open(dst)).get("kernels", {})
        for case, d in old.items():
            if case not in kernels:
                d.setdefault("captured", "earlier capture of this round (previous build)")
                kernels[case] = d
    with open(dst, "w") as f:
        json.dump(out, f, indent=1)
    print(dst, len(kernels), "kernels")
    # the bench's traffic lookup (roofline.traffic): dram read + write of the dominant kernel per launch
    bench_sum = {"source": dst, "kernels": {}}
    for case, d in kernels.items():
        bench_sum["kernels"][case.replace("square", "square_")] = {
            "dram_bytes": d.get("dram_read_B", 0) + d.get("dram_write_B", 0), "dram_read_B": d.get("dram_read_B"),
            "dram_write_B": d.get("dram_write_B"), "duration_us_ncu": d.get("duration_us")}
    with open(os.path.join(ROOT, "profiles", "ncu_bench_summary.json"), "w") as f:
        json.dump(bench_sum, f, indent=1)
    # launch list of the headline step
    lst = os.path.join(a.src, "launches_step.csv")
    if os.path.exists(lst):
        lines = [l for l in open(lst) if l.startswith('"')]
        rows = list(csv.reader(lines))
        hdr = rows[0]
        ki, mi, ui, vi, ii = (hdr.index(c) for c in ("Kernel Name", "Metric Name", "Metric Unit", "Metric Value", "ID"))
        per = {}
        for r in rows[1:]:
            d = per.setdefault(int(r[ii]), {"kernel": r[ki].split("(")[0].replace("void ", "")})
            d[r[mi]] = float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1)
        ids = sorted(per)
        seq = []
        for j, i in enumerate(ids):
            n = W.SQUARES[j % len(W.SQUARES)]
            seq.append({"square": n, "us": round(per[i].get("gpu__time_duration.sum", 0), 1),
                        "dram_read_MB": round(per[i].get("dram__bytes_read.sum", 0) / 1e6, 1),
                        "dram_write_MB": round(per[i].get("dram__bytes_write.sum", 0) / 1e6, 1),
                        "l2_write_MB": round(per[i].get("lts__t_sectors_op_write.sum", 0) / 1e6, 1),
                        "sm_mhz": round(per[i].get("sm__cycles_elapsed.avg.per_second", 0), 0)})
        tot = sum(s["us"] for s in seq)
        share = {}
        for s in seq:
            share[s["square"]] = share.get(s["square"], 0) + s["us"] / tot
        dst2 = os.path.join(ROOT, "profiles", "launches_step_%s.json" % a.round)
        with open(dst2, "w") as f:
            json.dump({"source": "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,"
                                 "lts__t_sectors_op_write.sum,sm__cycles_elapsed.avg.per_second --clock-control none "
                                 "-k regex:alcop python tools/profile_kernels.py step --reps 4 (serialized)",
                       "share_of_step": {str(k): round(v, 3) for k, v in share.items()}, "launches": seq}, f, indent=1)
        print(dst2, len(seq), "launches")


if __name__ == "__main__":
    main()
