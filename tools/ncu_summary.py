"""Summarise ncu output of tools/profile_step.py into profiles/ (measurement tool).

  python tools/ncu_summary.py launches <ncu --csv metrics log> <out.json>
  python tools/ncu_summary.py full <ncu -i rep --page raw --csv output> <out.json> [bench summary out]

Launches are labelled in profile_step's order (qkv_proj, o_proj, ffn1, ffn2)."""
import csv
import json
import sys

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
from bench import BERT_GEMMS  # noqa: E402

NAMES = [g[0] for g in BERT_GEMMS]
SHAPES = {g[0]: g[1:] for g in BERT_GEMMS}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1, "usecond": 1, "ms": 1e3,
         "msecond": 1e3, "nsecond": 1e-3}


def rows_of(path):
    lines = [l for l in open(path) if l.startswith('"')]
    return list(csv.reader(lines))


def launches(path, out):
    rows = rows_of(path)
    hdr = rows[0]
    ki, mi, ui, vi, ii = (hdr.index(c) for c in ("Kernel Name", "Metric Name", "Metric Unit", "Metric Value", "ID"))
    per = {}
    for r in rows[1:]:
        if "alcop" not in r[ki]:
            continue
        d = per.setdefault(int(r[ii]), {"kernel": r[ki].split("(")[0].replace("void ", ""), "grid": r[hdr.index("Grid Size")]})
        d[r[mi]] = float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1)
    ids = sorted(per)
    agg = {}
    for j, i in enumerate(ids):
        name = NAMES[j % len(NAMES)]
        a = agg.setdefault(name, {"kernel": per[i]["kernel"], "grid": per[i]["grid"], "shape": SHAPES[name], "n": 0,
                                  "us": 0.0, "dram_read_B": 0.0, "dram_write_B": 0.0, "sm_ghz": 0.0})
        a["n"] += 1
        a["us"] += per[i].get("gpu__time_duration.sum", 0)
        a["dram_read_B"] += per[i].get("dram__bytes_read.sum", 0)
        a["dram_write_B"] += per[i].get("dram__bytes_write.sum", 0)
        a["sm_ghz"] += per[i].get("sm__cycles_elapsed.avg.per_second", 0) / 1e3 if per[i].get("sm__cycles_elapsed.avg.per_second", 0) > 1e3 else per[i].get("sm__cycles_elapsed.avg.per_second", 0)
    tot = sum(a["us"] for a in agg.values())
    res = {}
    for name, a in agg.items():
        n = a["n"]
        M, N, K = a["shape"]
        res[name] = {"kernel": a["kernel"], "grid": a["grid"], "shape": a["shape"], "launches": n,
                     "mean_us": round(a["us"] / n, 2), "share": round(a["us"] / tot, 3),
                     "tflops_ncu": round(2.0 * M * N * K / (a["us"] / n) / 1e6, 1),
                     "dram_read_MB": round(a["dram_read_B"] / n / 1e6, 2),
                     "dram_write_MB": round(a["dram_write_B"] / n / 1e6, 2),
                     "algorithmic_MB": round((M * K + K * N + M * N) * 2 / 1e6, 2)}
    with open(out, "w") as f:
        json.dump({"source": "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                             "--clock-control none -k regex:alcop python tools/profile_step.py (plain launches, "
                             "serialized by ncu: compare shares, not absolutes)", "kernels": res}, f, indent=1)
    print(json.dumps(res, indent=1))


def full(path, out, bench_out=None):
    rows = rows_of(path)
    hdr, units = rows[0], rows[1]
    keep = ["Kernel Name", "Grid Size", "Block Size", "gpu__time_duration.sum", "dram__bytes_read.sum",
            "dram__bytes_write.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
            "lts__throughput.avg.pct_of_peak_sustained_elapsed", "sm__cycles_elapsed.avg.per_second",
            "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
            "l1tex__m_xbar2l1tex_read_bytes.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "dram__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"]
    idx = {k: hdr.index(k) for k in keep if k in hdr}
    caps = []
    for j, r in enumerate(rows[2:]):
        d = {k: r[i] for k, i in idx.items()}
        d["units"] = {k: units[i] for k, i in idx.items()}
        d["label"] = NAMES[j % len(NAMES)]
        caps.append(d)
    with open(out, "w") as f:
        json.dump({"source": "ncu --set full --clock-control none --import-source on -k regex:alcop "
                             "python tools/profile_step.py (one step: qkv_proj, o_proj, ffn1, ffn2)",
                   "captures": caps}, f, indent=1)
    if bench_out:
        def num(d, k):
            return float(d[k].replace(",", "")) * SCALE.get(d["units"][k], 1)
        kern = {}
        for d in caps:
            M, N, K = SHAPES[d["label"]]
            kern[d["label"]] = {
                "dram_bytes": int(num(d, "dram__bytes_read.sum") + num(d, "dram__bytes_write.sum")),
                "l2_to_sm_bytes": int(num(d, "l1tex__m_xbar2l1tex_read_bytes.sum")),
                "ncu_duration_us": round(num(d, "gpu__time_duration.sum"), 2),
                "tensor_pipe_active_pct": round(float(d["sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"]), 1),
                "sm_clock_ghz": d.get("sm__cycles_elapsed.avg.per_second"),
                "algorithmic_bytes": (M * K + K * N + M * N) * 2, "algorithmic_flops": 2 * M * N * K}
        with open(bench_out, "w") as f:
            json.dump({"source": out + " (ncu --set full, one bench step, cold inputs, serialized)",
                       "note": "dram bytes per launch = read + write from ncu", "kernels": kern}, f, indent=1)
    print(json.dumps(caps, indent=1)[:3000])


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        full(sys.argv[2], sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else None)
