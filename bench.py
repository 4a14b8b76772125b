#!/usr/bin/env python
"""bench.py — headline benchmark of the B200 pipelined load-and-use GEMM path.

Workload (BASELINE.json configs[1]): the GEMMs of one BERT-base encoder layer
at M = 4096 tokens, bf16 in / bf16 out, fp32 accumulate:
    Q, K, V projections     [4096 x 768] @ [768 x 2304]  (one GEMM: the three
                            projections read the same activations, so their
                            weights are stored side by side, B = [Wq|Wk|Wv])
    O projection            [4096 x 768]  @ [768 x 768]
    FFN1                    [4096 x 768]  @ [768 x 3072]
    FFN2                    [4096 x 3072] @ [3072 x 768]
(--unfused-qkv: Q, K, V as three [768 x 768] GEMMs; the same FLOPs, six
launches; that variant's step time is reported beside the headline too.)
B is the reference layout [K, N] row-major (schedule.hpp:389).  One "step" is
one pass over those GEMMs, each launched through the C ABI (alcop_gemm)
with the schedule alcop_tune picks (the analytical model's top schedules
timed on this GPU; --schedule model: the model's first pick).  Inputs
rotate over copies whose footprint exceeds 2x the 126 MB L2, so every step
reads HBM.  Reported beside it, in the same run: the n_stage 1..6 sweep of
each distinct shape (speedup vs the non-pipelined n_stage=1 variant), the
model pick vs the best swept schedule, BASELINE config 1 (fp16 512^3 with the
reference's own schedule script, and the reference interpreter on the whole
problem on the host cores), the attention BMMs, the ResNet-50 convs, the
large square GEMMs, the roofline of
the dominant kernel, the end-to-end number through the host-buffer ABI entry
point, and the reference CPU path timed on the host cores.

--impl reference times the reference's own CPU implementation (the pipec
interpreter running the transformed program, oracle/_ref/ref_driver built
from /root/reference) on a bounded sample of the same workload.

Multi-GPU: the BERT GEMMs are replicas only — each rank runs
the full step on its own GPU, no collective on the data path; value is the
whole-job FLOP rate (N x per-GPU FLOPs / max-over-ranks time).
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

BERT_GEMMS = [  # (name, M, N, K): the layer's GEMMs, Q/K/V fused into one launch
    ("qkv_proj", 4096, 2304, 768), ("o_proj", 4096, 768, 768), ("ffn1", 4096, 3072, 768),
    ("ffn2", 4096, 768, 3072),
]
BERT_GEMMS_UNFUSED = [
    ("q_proj", 4096, 768, 768), ("k_proj", 4096, 768, 768), ("v_proj", 4096, 768, 768),
    ("o_proj", 4096, 768, 768), ("ffn1", 4096, 3072, 768), ("ffn2", 4096, 768, 3072),
]
METRIC = "TFLOP/s (BERT-base layer GEMMs, M=4096, bf16)"
# ResNet-50 v1.5 convolutions at batch 256 (BASELINE configs[3]); conv1 (C=3) runs
# the stem kernel on the NHWC8 halo-padded input.
# (name, H_in, C, K, R, stride, pad, repeats)
RESNET50_CONVS = [
    ("conv1_7x7s2_3_64", 224, 3, 64, 7, 2, 3, 1),  # NHWC input padded to 8 channels (zero filter taps)
    ("l1_1x1_64_64", 56, 64, 64, 1, 1, 0, 1), ("l1_3x3_64_64", 56, 64, 64, 3, 1, 1, 3),
    ("l1_1x1_64_256", 56, 64, 256, 1, 1, 0, 4), ("l1_1x1_256_64", 56, 256, 64, 1, 1, 0, 2),
    ("l2_1x1_256_128", 56, 256, 128, 1, 1, 0, 1), ("l2_3x3s2_128", 56, 128, 128, 3, 2, 1, 1),
    ("l2_3x3_128", 28, 128, 128, 3, 1, 1, 3), ("l2_1x1_128_512", 28, 128, 512, 1, 1, 0, 4),
    ("l2_ds_256_512", 56, 256, 512, 1, 2, 0, 1), ("l2_1x1_512_128", 28, 512, 128, 1, 1, 0, 3),
    ("l3_1x1_512_256", 28, 512, 256, 1, 1, 0, 1), ("l3_3x3s2_256", 28, 256, 256, 3, 2, 1, 1),
    ("l3_3x3_256", 14, 256, 256, 3, 1, 1, 5), ("l3_1x1_256_1024", 14, 256, 1024, 1, 1, 0, 6),
    ("l3_ds_512_1024", 28, 512, 1024, 1, 2, 0, 1), ("l3_1x1_1024_256", 14, 1024, 256, 1, 1, 0, 5),
    ("l4_1x1_1024_512", 14, 1024, 512, 1, 1, 0, 1), ("l4_3x3s2_512", 14, 512, 512, 3, 2, 1, 1),
    ("l4_3x3_512", 7, 512, 512, 3, 1, 1, 2), ("l4_1x1_512_2048", 7, 512, 2048, 1, 1, 0, 3),
    ("l4_ds_1024_2048", 14, 1024, 2048, 1, 2, 0, 1), ("l4_1x1_2048_512", 7, 2048, 512, 1, 1, 0, 2),
]
UNIT = "TFLOP/s"
TUNE_BUDGET = 24
L2_BYTES = 126 * 1024 * 1024


def step_flops():
    return sum(2.0 * M * N * K for _, M, N, K in BERT_GEMMS)


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return {"bf16_tflops": d["bf16_tflops"], "bf16_tflops_sustained": d["bf16_tflops_sustained"],
                "hbm_gbs": d["hbm_gbs"], "source": "measured"}
    return {"bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "hbm_gbs": 6650.0, "source": "fallback"}


# ----------------------------------------------------------------- CPU arms
def _ref_driver():
    p = os.path.join(ROOT, "oracle", "_ref", "ref_driver")
    return p if os.path.exists(p) else None


REF_SAMPLE_COLS = 128  # one output sub-block per GEMM: rows x 128 columns, full K
REF_NS_PER_MMA = 150e-9  # measured cost of one interpreted mma statement


def ref_sample_rows(seconds_per_step):
    """Rows of the sample block so the slowest job (FFN2, K=3072) takes ~seconds_per_step."""
    kmax = max(K for _, _, _, K in BERT_GEMMS)
    return max(1, min(128, int(seconds_per_step / (REF_NS_PER_MMA * REF_SAMPLE_COLS * kmax))))


def _ref_sample_script(M, N, K):
    # the reference's own config-1-style schedule for the sample block:
    # one output tile, tileK = 32, 2-stage shared + 2-stage register pipeline
    ko = K // 32
    return ("cache_read A shared\ncache_read B shared\ncache_read A_shared register\n"
            "cache_read B_shared register\ntile C i0=1 i1=%d j0=1 j1=%d ko=%d ki=32\n"
            "pipeline A_shared 2\npipeline B_shared 2\npipeline A_reg 2\npipeline B_reg 2\n"
            % (M, N, ko))


def cpu_reference_step(rows):
    """One step of the reference CPU path on a bounded sample: for every GEMM
    of the layer, a rows x REF_SAMPLE_COLS output block per process with the
    full K, interpreted by the reference (pipec::run on the transformed
    program); max(#GEMMs, host cores) processes run concurrently, the GEMMs
    dealt round-robin, so every host core works (the interpreter is
    single-threaded per run and runs are independent).
    Returns (seconds, flops, kind, cores).  Each block is a sub-problem of the
    same GEMM: the interpreter's cost is linear in rows*cols*K."""
    import tempfile
    drv = _ref_driver()
    jobs = []
    tmp = tempfile.mkdtemp()
    nproc = max(len(BERT_GEMMS), os.cpu_count() or 1)
    for j in range(nproc):
        name, M, N, K = BERT_GEMMS[j % len(BERT_GEMMS)]
        m, n = rows, REF_SAMPLE_COLS
        sp = os.path.join(tmp, "%s_%d.txt" % (name, j))
        with open(sp, "w") as f:
            f.write(_ref_sample_script(m, n, K))
        jobs.append((name, m, n, K, sp))
    flops = sum(2.0 * m * n * K for _, m, n, K, _ in jobs)
    cores = os.cpu_count() or 1
    if drv is not None:
        t0 = time.perf_counter()
        ps = [subprocess.Popen([drv, "time", "--M", str(m), "--N", str(n), "--K", str(K), "--script", sp,
                                "--mode", "stale"], stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)
              for _, m, n, K, sp in jobs]
        outs = [p.communicate() for p in ps]
        dt = time.perf_counter() - t0
        for p, (o, e) in zip(ps, outs):
            if p.returncode != 0:
                raise RuntimeError("ref_driver failed: " + e)
        return dt, flops, "reference", min(cores, len(jobs))
    # port: the oracle's C restatement (fp32-accumulate GEMM, OpenMP on all cores)
    import numpy as np
    from oracle import coracle
    t0 = time.perf_counter()
    for _, m, n, K, _ in jobs:
        A = coracle.to_dtype(np.ones((m, K), np.float32), "bf16")
        B = coracle.to_dtype(np.ones((K, n), np.float32), "bf16")
        coracle.gemm(A, B, "bf16", "bf16")
    return time.perf_counter() - t0, flops, "port", cores


def run_reference_arm(args, rank, world):
    if rank != 0:
        return
    times = []
    kind = cores = None
    flops = 0.0
    rows = ref_sample_rows(min(3.0, 150.0 / (args.warmup + args.steps)))
    for i in range(args.warmup + args.steps):
        dt, flops, kind, cores = cpu_reference_step(rows)
        if i >= args.warmup:
            times.append(dt)
    total = sum(times)
    value = flops * len(times) / total / 1e12
    sample = ("per step: %d concurrent processes (host cores), each a %dx%d output block (full K) of one of the %d "
              "BERT-layer GEMMs (round-robin), pipec::run on the transformed two-level program (tile %dx%dx32, "
              "2+2 stages)" % (max(len(BERT_GEMMS), os.cpu_count() or 1), rows, REF_SAMPLE_COLS, len(BERT_GEMMS),
                               rows, REF_SAMPLE_COLS))
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": total / len(times) * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int64",
            "data": "synthetic (SplitMix64 range(-8,8), the reference generator)",
            "config": {"workload": "bert_base_layer_gemms_sample", "M": 4096, "gemms": [g[1:] for g in BERT_GEMMS]},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind, "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------- clocks
class ClockSampler:
    """NVML sampling of SM clock and clocks-event reasons during the timed region."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}

    def __init__(self, device_index, period_s=0.005):
        self.samples = []
        self.reasons = 0
        self.max_mhz = None
        self.ok = False
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.nv = None
        self.period = period_s
        self.t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                try:
                    r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                except AttributeError:
                    r = self.nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                self.reasons |= int(r) & ~0x1
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": [n for b, n in self.REASONS.items() if self.reasons & b], "samples": len(self.samples)}


class _Null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


# ----------------------------------------------------------------- GPU arm
def main_gpu(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    import paper_2210_16691_b200 as alcop
    from paper_2210_16691_b200.timing import time_graph

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    alcop.load_library()
    peaks = load_peaks()
    stream = torch.cuda.current_stream()

    gemms = BERT_GEMMS_UNFUSED if args.unfused_qkv else BERT_GEMMS
    lib = alcop.load_library()
    import ctypes
    sp = ctypes.c_void_p(stream.cuda_stream)
    descs, sched = {}, {}

    model_pick = {}

    def plan(shape):
        # per distinct shape: the analytical model's ranking (alcop_choose_schedule);
        # with --schedule tune (default) its top TUNE_BUDGET schedules are timed on
        # this GPU and the fastest is used (alcop_tune: the reference's
        # model-assisted tuning, tuner.hpp:363-531, on real B200 timings)
        if shape not in sched:
            descs[shape] = alcop.gemm_desc(*shape, 1, alcop.BF16, alcop.BF16, alcop.B_KN)
            model_pick[shape] = alcop.choose_schedule(descs[shape])
            sched[shape] = model_pick[shape]
            if args.schedule == "tune":
                M, N, K = shape
                A = (torch.rand((M, K), device=dev) - 0.5).to(torch.bfloat16)
                B = (torch.rand((K, N), device=dev) - 0.5).to(torch.bfloat16)
                C = torch.empty((M, N), device=dev, dtype=torch.bfloat16)
                sched[shape], _ = alcop.tune(A, B, C, budget=TUNE_BUDGET)
                del A, B, C
        return sched[shape]

    def launch(A, B, C, s, shape):
        cur = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        rc = lib.alcop_gemm(ctypes.byref(descs[shape]), ctypes.byref(s), ctypes.c_void_p(A.data_ptr()),
                            ctypes.c_void_p(B.data_ptr()), ctypes.c_void_p(C.data_ptr()), cur)
        if rc:
            raise alcop.AlcopError(rc, lib.alcop_last_error().decode())

    g = torch.Generator(device=dev)
    g.manual_seed(1234 + rank)

    def make_step(gl):
        """CUDA graphs of one step over the GEMM list gl, one graph per input
        set; input sets rotate so the step's operands come from HBM (> 2x L2).
        The launches are chained with PDL (the kernels are unchanged)."""
        set_bytes = sum((M * K + K * N + M * N) * 2 for _, M, N, K in gl)
        nsets = max(2, -(-2 * L2_BYTES // set_bytes))
        sets = []
        for _ in range(nsets):
            one = []
            for name, M, N, K in gl:
                A = (torch.rand((M, K), generator=g, device=dev) * 2 - 1).to(torch.bfloat16)
                B = (torch.rand((K, N), generator=g, device=dev) * 2 - 1).to(torch.bfloat16)
                C = torch.empty((M, N), device=dev, dtype=torch.bfloat16)
                one.append((A, B, C, plan((M, N, K))))
            sets.append(one)

        def step_set(i):
            for (name, M, N, K), (A, B, C, s) in zip(gl, sets[i]):
                launch(A, B, C, s, (M, N, K))

        cs = torch.cuda.Stream()
        cs.wait_stream(stream)
        with torch.cuda.stream(cs):
            for i in range(nsets):
                step_set(i)
        stream.wait_stream(cs)
        torch.cuda.synchronize()
        use_graphs = os.environ.get("ALCOP_BENCH_GRAPHS", "1") != "0"  # 0: direct launches (profiling)
        graphs = []
        if use_graphs:
            for i in range(nsets):
                g_ = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g_):
                    step_set(i)
                graphs.append(g_)
        state = {"i": 0}

        def step():
            if use_graphs:
                graphs[state["i"]].replay()
            else:
                step_set(state["i"])
            state["i"] = (state["i"] + 1) % nsets
        return step, nsets, set_bytes

    def loaded_sm_clock(gl, iters=40):
        """Effective SM clock under this workload's load: CTA 0 of the step's
        last GEMM stamps clock64 and %globaltimer at start and end (debug
        stamps, alcop_debug_set_stamps) after `iters` back-to-back steps.
        NVML's SM clock reading does not show the loaded clock."""
        lib.alcop_debug_set_stamps.argtypes = [ctypes.c_void_p]
        buf = torch.zeros(148 * 8 + 64 + 128 + 2, dtype=torch.int64, device=dev)
        ins = []
        for name, M, N, K in gl:
            ins.append(((torch.rand((M, K), device=dev) - 0.5).to(torch.bfloat16),
                        (torch.rand((K, N), device=dev) - 0.5).to(torch.bfloat16),
                        torch.empty((M, N), device=dev, dtype=torch.bfloat16), (M, N, K)))
        torch.cuda.synchronize()
        lib.alcop_debug_set_stamps(ctypes.c_void_p(buf.data_ptr()))
        try:
            for _ in range(iters):
                for A, B, C, shape in ins:
                    launch(A, B, C, sched[shape], shape)
            torch.cuda.synchronize()
        finally:
            lib.alcop_debug_set_stamps(None)
        t = buf.cpu().tolist()
        ns = t[7] - t[0]
        cyc = t[148 * 8 + 193] - t[148 * 8 + 192]
        return round(cyc / ns * 1e3) if ns > 0 and cyc > 0 else None

    step, nsets, set_bytes = make_step(gemms)
    shapes = sorted(set((M, N, K) for _, M, N, K in gemms))

    def barrier():
        if world > 1:
            dist.barrier()

    # ---- correctness spot check of this run's kernels (oracle-independent: exact-integer inputs)
    for (M, N, K) in shapes:
        a = torch.randint(-8, 9, (M, K), device=dev).to(torch.bfloat16)
        b = torch.randint(-8, 9, (K, N), device=dev).to(torch.bfloat16)
        c = torch.empty((M, N), device=dev, dtype=torch.float32)
        d32 = alcop.gemm_desc(M, N, K, 1, alcop.BF16, alcop.F32, alcop.B_KN)
        rc = lib.alcop_gemm(ctypes.byref(d32), ctypes.byref(sched[(M, N, K)]), ctypes.c_void_p(a.data_ptr()),
                            ctypes.c_void_p(b.data_ptr()), ctypes.c_void_p(c.data_ptr()), sp)
        assert rc == 0
        ref = (a.double() @ b.double()).float()
        assert torch.equal(c, ref), "kernel mismatch on %s" % ((M, N, K),)

    def timed(stepfn, steps, sample_clocks=False):
        for _ in range(args.warmup):
            stepfn()
        torch.cuda.synchronize()
        barrier()
        torch.cuda.synchronize()
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        with ClockSampler(local_rank) if sample_clocks else _Null() as clk:
            ev0.record(stream)
            for _ in range(steps):
                stepfn()
            ev1.record(stream)
            torch.cuda.synchronize()
        ms_total = ev0.elapsed_time(ev1)
        barrier()
        t = torch.tensor([ms_total], device=dev, dtype=torch.float64)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item()), clk

    # ---- warmup + timed region (the headline)
    ms_max, clk = timed(step, args.steps, sample_clocks=True)
    kclk = loaded_sm_clock(gemms)
    flops = step_flops()
    value = world * flops * args.steps / (ms_max * 1e-3) / 1e12
    # the other decomposition of the same layer (same FLOPs), same run
    alt_gemms = BERT_GEMMS if args.unfused_qkv else BERT_GEMMS_UNFUSED
    alt_step, _, _ = make_step(alt_gemms)
    alt_steps = max(50, args.steps // 4)
    alt_ms, _ = timed(alt_step, alt_steps)
    alt = {"gemms": {n: [M, N, K] for n, M, N, K in alt_gemms}, "launches_per_step": len(alt_gemms),
           "ms_per_step": alt_ms / alt_steps, "tflops": world * flops * alt_steps / (alt_ms * 1e-3) / 1e12}
    del alt_step
    torch.cuda.empty_cache()
    # the same GEMMs as ONE persistent launch (alcop_gemm_chain): the smem and
    # TMEM rings never drain between GEMMs; with row-block dependencies
    # (A_p row block waits for C_{p-1} row block: the layer order) and as
    # independent GEMMs (grouped launch, no ordering)
    chain = {}
    if not args.unfused_qkv:
        csets = [[((torch.rand((M, K), device=dev) - 0.5).to(torch.bfloat16),
                   (torch.rand((K, N), device=dev) - 0.5).to(torch.bfloat16),
                   torch.empty((M, N), device=dev, dtype=torch.bfloat16)) for _, M, N, K in gemms]
                 for _ in range(nsets)]
        cws = torch.empty(1 << 16, dtype=torch.uint8, device=dev)
        for label, dep in (("row_block_dependencies", [0] + [1] * (len(gemms) - 1)), ("independent", None)):
            best = None
            for tn, tk, st in ((192, 64, 5), (256, 64, 4), (128, 128, 3)):
                cs_ = alcop.make_schedule(tileN=tn, tileK=tk, n_stage=st)
                ms = time_graph(lambda i: alcop.gemm_chain(csets[i % nsets], cs_, dep=dep, workspace=cws),
                                iters=max(30, 6 * nsets), reps_per_graph=nsets)
                if best is None or ms < best[0]:
                    best = (ms, cs_)
            tt = torch.tensor([best[0]], device=dev, dtype=torch.float64)
            if world > 1:
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            chain[label] = {"us_per_step": round(float(tt.item()) * 1e3, 2),
                            "tflops": round(world * flops / (float(tt.item()) * 1e-3) / 1e12, 1),
                            "schedule": best[1].as_dict()}
        del csets
        torch.cuda.empty_cache()

    # ---- per-GEMM times (CUDA graphs on the launching stream, each GEMM on its
    # own rotating inputs > 2x L2, i.e. cold operands as inside the step)
    per = {}
    reps = max(8, min(50, args.steps // 4))
    from paper_2210_16691_b200.timing import Rotating
    for (name, M, N, K) in gemms:
        if (M, N, K) in [tuple(v["shape"]) for v in per.values()]:
            continue
        rot = Rotating(lambda i, M=M, N=N, K=K: ((torch.rand((M, K), device=dev) - 0.5).to(torch.bfloat16),
                                                 (torch.rand((K, N), device=dev) - 0.5).to(torch.bfloat16),
                                                 torch.empty((M, N), device=dev, dtype=torch.bfloat16)),
                       (M * K + K * N + M * N) * 2, max_sets=16)
        nr = len(rot.sets)

        def one(i, rot=rot, nr=nr, M=M, N=N, K=K):
            A, B, C = rot.sets[i % nr]
            launch(A, B, C, sched[(M, N, K)], (M, N, K))
        ms = time_graph(one, iters=max(reps, 2 * nr), warmup=3, reps_per_graph=nr)
        per[name] = {"ms": ms, "shape": [M, N, K], "tflops": 2.0 * M * N * K / (ms * 1e-3) / 1e12,
                     "schedule": sched[(M, N, K)].as_dict()}
        del rot
    count = {}
    for (name, M, N, K) in gemms:
        key = [n for n, v in per.items() if v["shape"] == [M, N, K]][0]
        count[key] = count.get(key, 0) + 1
    step_ms_est = sum(per[n]["ms"] * c for n, c in count.items())
    dom = max(per, key=lambda n: per[n]["ms"] * count[n])
    dM, dN, dK = per[dom]["shape"]
    dflops = 2.0 * dM * dN * dK
    achieved = dflops / (per[dom]["ms"] * 1e-3) / 1e12
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_bench_summary.json")
    if os.path.exists(prof):
        try:
            with open(prof) as f:
                pj = json.load(f)
            traffic = pj.get("kernels", {}).get(dom, {}).get("dram_bytes")
        except Exception:
            traffic = None
    roofline = {"bound": "tensor", "achieved": achieved, "peak": peaks["bf16_tflops"], "unit": "TFLOP/s",
                "frac": achieved / peaks["bf16_tflops"], "traffic": traffic,
                "kernel": "alcop_pipelined_gemm_kernel (%s %dx%dx%d)" % (dom, dM, dN, dK),
                "share_of_step": per[dom]["ms"] * count[dom] / step_ms_est,
                "peak_source": peaks["source"] + " burst bf16 (MEASURED_PEAKS.json)",
                "algorithmic_flops_per_launch": dflops,
                "timing": "CUDA events around CUDA graphs of this GEMM alone, rotating cold inputs > 2x L2"}

    def attainable(fl, byts):
        """min(P, AI * BW) in TFLOP/s, AI = FLOPs / compulsory bytes."""
        return min(peaks["bf16_tflops"], fl / byts * peaks["hbm_gbs"] * 1e-3)

    def config1_block():
        """BASELINE configs[0]: fp16 512^3 with the reference's
        own schedule script (tile 128x128x32, 2 shared + 2 register stages)
        mapped through alcop_parse_schedule_script, in WRAP (the pass's exact
        index algebra) and FUSED mode, plus the model pick; L2 flushed between
        launches (rotating inputs > 2x L2).  Beside it, on this host: the
        reference interpreter on the WHOLE C1 problem (its 16 output tiles as
        concurrent processes; makespan) and the C oracle (OpenMP)."""
        M = N = K = 512
        d1 = alcop.gemm_desc(M, N, K, 1, alcop.F16, alcop.F16, alcop.B_KN)
        script = _ref_sample_script(128, 128, K).replace("i0=1", "i0=%d" % (M // 128)).replace(
            "j0=1", "j0=%d" % (N // 128))
        s_ref, _ = alcop.apply_script(d1, script)
        s_fused = alcop.Schedule.from_buffer_copy(s_ref)
        s_fused.mode = alcop.MODE_FUSED
        s_model = alcop.choose_schedule(d1)
        rot = Rotating(lambda i: ((torch.rand((M, K), device=dev) - 0.5).to(torch.float16),
                                  (torch.rand((K, N), device=dev) - 0.5).to(torch.float16),
                                  torch.empty((M, N), device=dev, dtype=torch.float16)),
                       (M * K + K * N + M * N) * 2, max_sets=192)
        nr = len(rot.sets)

        def run1(i, s_):
            A, B, C = rot.sets[i % nr]
            rc = lib.alcop_gemm(ctypes.byref(d1), ctypes.byref(s_), ctypes.c_void_p(A.data_ptr()),
                                ctypes.c_void_p(B.data_ptr()), ctypes.c_void_p(C.data_ptr()),
                                ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
            if rc:
                raise alcop.AlcopError(rc, lib.alcop_last_error().decode())
        out = {"shape": [M, N, K], "dtype": "f16", "script": script.strip().split("\n"),
               "l2": "flushed (%d rotating input sets)" % nr}
        fl = 2.0 * M * N * K
        for label, s_ in (("reference_schedule_wrap", s_ref), ("reference_schedule_fused", s_fused),
                          ("model_pick", s_model)):
            ms = time_graph(lambda i, s_=s_: run1(i, s_), iters=2 * nr, warmup=3, reps_per_graph=nr)
            out[label] = {"us": round(ms * 1e3, 2), "tflops": round(fl / (ms * 1e-3) / 1e12, 1),
                          "schedule": s_.as_dict()}
        del rot
        if args.no_cpu:
            return out
        import tempfile
        drv = _ref_driver()
        if drv is not None:
            sp = os.path.join(tempfile.mkdtemp(), "c1_tile.txt")
            with open(sp, "w") as f:
                f.write(_ref_sample_script(128, 128, K))
            t0 = time.perf_counter()
            ps = [subprocess.Popen([drv, "time", "--M", "128", "--N", "128", "--K", str(K), "--script", sp,
                                    "--mode", "stale", "--seed", str(t)], stdout=subprocess.PIPE,
                                   stderr=subprocess.PIPE, text=True) for t in range((M // 128) * (N // 128))]
            outs = [p.communicate() for p in ps]
            dt = time.perf_counter() - t0
            if all(p.returncode == 0 for p in ps):
                run_s = [json.loads(o.strip().splitlines()[-1])["best_s"] for o, _ in outs]
                out["cpu_reference"] = {
                    "makespan_s": round(dt, 3), "sum_of_run_s": round(sum(run_s), 2),
                    "processes": len(ps), "host_cores": os.cpu_count(),
                    "what": "pipec::run on transform(lower(apply_script(...))) of each 128x128 output tile "
                            "(full K, the config-1 script), 16 concurrent processes = the whole C1 problem"}
                best_us = min(out[k]["us"] for k in ("reference_schedule_wrap", "reference_schedule_fused",
                                                     "model_pick"))
                out["gpu_speedup_vs_cpu_reference"] = round(dt / (best_us * 1e-6), 0)
        import numpy as np
        from oracle import coracle
        A = coracle.to_dtype(np.ones((M, K), np.float32), "f16")
        B = coracle.to_dtype(np.ones((K, N), np.float32), "f16")
        coracle.gemm(A, B, "f16", "f16")
        t0 = time.perf_counter()
        for _ in range(3):
            coracle.gemm(A, B, "f16", "f16")
        out["cpu_oracle_openmp_s"] = round((time.perf_counter() - t0) / 3, 4)
        return out

    extra = {}
    if rank == 0 and not args.quick:
        # ---- n_stage sweep 1..5 per distinct shape (same tile, same run) + model pick vs best
        sweep = {}
        for (M, N, K) in shapes:
            base = model_pick[(M, N, K)]
            tuned = sched[(M, N, K)]
            rows = []
            rot = Rotating(lambda i, M=M, N=N, K=K: ((torch.rand((M, K), device=dev) - 0.5).to(torch.bfloat16),
                                                     (torch.rand((K, N), device=dev) - 0.5).to(torch.bfloat16),
                                                     torch.empty((M, N), device=dev, dtype=torch.bfloat16)),
                           (M * K + K * N + M * N) * 2, max_sets=16)
            nr = len(rot.sets)

            def run_on(i, s, rot=rot, nr=nr, M=M, N=N, K=K):
                A, B, C = rot.sets[i % nr]
                launch(A, B, C, s, (M, N, K))
            best = None
            cands = []
            for st in range(1, 7):
                for tn, tk, cg in ((base.tileN, base.tileK, base.cta_group), (128, 64, 1), (256, 64, 1),
                                   (128, 128, 1), (256, 128, 1), (192, 64, 1), (256, 64, 2), (128, 64, 2)):
                    s = alcop.make_schedule(tileN=tn, tileK=tk, n_stage=st, n_stage_inner=2 if st > 1 else 1,
                                            cta_group=cg)
                    try:
                        alcop.validate(descs[(M, N, K)], s)
                    except alcop.AlcopError:
                        continue
                    cands.append((st, tn, tk, cg, s))
            for st, tn, tk, cg, s in cands:
                ms = time_graph(lambda i, s=s: run_on(i, s), iters=2 * nr, warmup=3, reps_per_graph=nr)
                tf = 2.0 * M * N * K / (ms * 1e-3) / 1e12
                rows.append({"n_stage": st, "tileN": tn, "tileK": tk, "cta_group": cg, "tflops": round(tf, 1)})
                if best is None or tf > best[0]:
                    best = (tf, st, tn, tk, cg)
            ms_pick = time_graph(lambda i: run_on(i, base), iters=2 * nr, warmup=3, reps_per_graph=nr)
            tf_pick = 2.0 * M * N * K / (ms_pick * 1e-3) / 1e12
            ms_tuned = time_graph(lambda i: run_on(i, tuned), iters=2 * nr, warmup=3, reps_per_graph=nr)
            tf_tuned = 2.0 * M * N * K / (ms_tuned * 1e-3) / 1e12
            by_stage = {}
            for r in rows:
                if (r["tileN"], r["tileK"], r["cta_group"]) == (base.tileN, base.tileK, base.cta_group):
                    by_stage[r["n_stage"]] = max(by_stage.get(r["n_stage"], 0), r["tflops"])
            s1 = max([r["tflops"] for r in rows if r["n_stage"] == 1] or [float("nan")])
            sweep["%dx%dx%d" % (M, N, K)] = {
                "tflops_by_n_stage_model_tile": by_stage,
                "best_n_stage1_tflops": s1,
                "best_swept": {"tflops": round(best[0], 1), "n_stage": best[1], "tileN": best[2], "tileK": best[3],
                               "cta_group": best[4]},
                "model_pick": {"tflops": round(tf_pick, 1), **{k: v for k, v in base.as_dict().items()
                                                              if k in ("tileN", "tileK", "n_stage_smem_A",
                                                                       "cta_group")}},
                "model_pick_over_best_time": round(best[0] / tf_pick, 3),
                "tuned_pick": {"tflops": round(tf_tuned, 1), **{k: v for k, v in tuned.as_dict().items()
                                                               if k in ("tileN", "tileK", "n_stage_smem_A",
                                                                        "cta_group")}},
                "speedup_best_vs_n_stage1": round(best[0] / s1, 2)}
        extra["n_stage_sweep"] = sweep
    if not args.quick:
        # ---- batched GEMMs of attention (BASELINE configs[2]): batch*heads = 192,
        # seq 512, head_dim 64; QK^T [512x64]@[64x512], PV [512x512]@[512x64];
        # HBM-bound (AI ~51 FLOP/B), batch-sharded across ranks
        bmm = {}
        from paper_2210_16691_b200.sharded import shard_range
        nb = shard_range(192, rank, world).size
        for name, (M, N, K) in (("qk_t", (512, 512, 64)), ("pv", (512, 64, 512))):
            db = alcop.gemm_desc(M, N, K, nb, alcop.BF16, alcop.BF16, alcop.B_KN)
            descs[("bmm", name)] = db
            sb = alcop.choose_schedule(db)
            rot = Rotating(lambda i, M=M, N=N, K=K: ((torch.rand((nb, M, K), device=dev) - 0.5).to(torch.bfloat16),
                                                     (torch.rand((nb, K, N), device=dev) - 0.5).to(torch.bfloat16),
                                                     torch.empty((nb, M, N), device=dev, dtype=torch.bfloat16)),
                           (M * K + K * N + M * N) * 2 * nb, max_sets=16)
            nr = len(rot.sets)
            if args.schedule == "tune":  # as for the layer GEMMs: the model's top schedules timed here
                sb, _ = alcop.tune(*rot.sets[0], budget=TUNE_BUDGET)

            def runb(i, s_, rot=rot, nr=nr, db=db):
                A, B, C = rot.sets[i % nr]
                rc = lib.alcop_gemm(ctypes.byref(db), ctypes.byref(s_), ctypes.c_void_p(A.data_ptr()),
                                    ctypes.c_void_p(B.data_ptr()), ctypes.c_void_p(C.data_ptr()),
                                    ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
                if rc:
                    raise alcop.AlcopError(rc, lib.alcop_last_error().decode())
            ms = time_graph(lambda i: runb(i, sb), iters=12 * nr, warmup=3, reps_per_graph=nr)
            s1 = alcop.make_schedule(tileN=sb.tileN, tileK=sb.tileK, n_stage=1, n_stage_inner=1)
            ms1 = time_graph(lambda i: runb(i, s1), iters=6 * nr, warmup=3, reps_per_graph=nr)
            tt = torch.tensor([ms], device=dev, dtype=torch.float64)
            if world > 1:
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            byts = (M * K + K * N + M * N) * 2 * 192
            tsec = float(tt.item()) * 1e-3
            bmm[name] = {"shape": [M, N, K], "batch": 192, "tflops_aggregate": round(2.0 * M * N * K * 192 / tsec / 1e12, 1),
                         "gbs_aggregate": round(byts / tsec / 1e9, 1),
                         "hbm_frac_per_gpu": round(byts / tsec / 1e9 / world / peaks["hbm_gbs"], 3),
                         "speedup_vs_n_stage1": round(ms1 / ms, 2), "schedule": sb.as_dict()}
            del rot
        extra["bmm_attention"] = {"sharding": "batch", "bound": "hbm", "gemms": bmm}
        if rank == 0:
            extra["config1_512"] = config1_block()

    # ---- ResNet-50 implicit-GEMM convs, batch 256 sharded across ranks
    if not args.quick:
        from paper_2210_16691_b200.sharded import shard_range
        sh = shard_range(256, rank, world)
        nloc = sh.size
        conv_rows = []
        tot_flops = 0.0
        tot_ms = 0.0
        for (name, H, C, K, R, st, pd, rep) in RESNET50_CONVS:
            P, Q = alcop.conv_out_hw(H, H, R, R, (st, st), (pd, pd))
            Cs = -(-C // 8) * 8  # stored channels (conv1: 3 -> 8, zero padded)
            halo = R * Cs <= 64  # stem layer: network input stored with its padding halo (NHWC8)
            hp = pd if halo else 0
            g = alcop.gemm_desc(nloc * P * Q, K, R * 64 if halo else R * R * Cs, 1, alcop.BF16, alcop.BF16,
                                alcop.B_NK)
            cs = alcop.choose_conv_schedule(g)
            X = torch.zeros((nloc, H + 2 * hp, H + 2 * hp, Cs), device=dev, dtype=torch.bfloat16)
            Wf = torch.zeros((K, R, R, Cs), device=dev, dtype=torch.bfloat16)
            X[:, hp:hp + H, hp:hp + H, :C] = (torch.rand((nloc, H, H, C), device=dev) - 0.5).to(torch.bfloat16)
            Wf[..., :C] = (torch.rand((K, R, R, C), device=dev) - 0.5).to(torch.bfloat16)
            Y = torch.empty((nloc, P, Q, K), device=dev, dtype=torch.bfloat16)
            ms = time_graph(lambda i: alcop.conv2d(X, Wf, (st, st), (pd, pd), sched=cs, out=Y, x_halo=halo),
                            iters=6, warmup=2)
            s1 = alcop.make_schedule(tileN=cs.tileN, tileK=64, n_stage=1, n_stage_inner=1)
            ms1 = time_graph(lambda i: alcop.conv2d(X, Wf, (st, st), (pd, pd), sched=s1, out=Y, x_halo=halo),
                             iters=4, warmup=1)
            fl = 2.0 * nloc * P * Q * K * R * R * C
            tot_flops += fl * rep
            tot_ms += ms * rep
            cbytes = 2 * (nloc * H * H * C + K * R * R * C + nloc * P * Q * K)
            conv_rows.append({"layer": name, "tflops": round(fl / (ms * 1e-3) / 1e12, 1),
                              "frac_of_attainable": round(fl / (ms * 1e-3) / 1e12 / attainable(fl, cbytes), 3),
                              "speedup_vs_n_stage1": round(ms1 / ms, 2), "tileN": cs.tileN,
                              "n_stage": cs.n_stage_smem_A})
            del X, Wf, Y
        tt = torch.tensor([tot_ms], device=dev, dtype=torch.float64)
        if world > 1:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        extra["resnet50_convs_b256"] = {
            "tflops_aggregate": round(world * tot_flops / (float(tt.item()) * 1e-3) / 1e12, 1),
            "images_per_gpu": nloc, "sharding": "batch", "layers": conv_rows,
            "note": "sum over all 53 conv layers (conv1: stem kernel on the NHWC8 halo-padded input, C 3 -> 8 "
                    "zero-padded, FLOPs counted at C=3); "
                    "per-layer CUDA-graph timing, model schedules"}
        torch.cuda.empty_cache()
        # ---- large square GEMMs (BASELINE configs[4]): n^3 bf16, n = 4096..16384,
        # M-sharded across ranks (rows of A and C split in 256-row granules, B
        # replicated, no collective on the compute path); aggregate =
        # total FLOPs / max-over-ranks time.  At N > 1 the optional NCCL
        # all-gather of C is timed separately.
        from paper_2210_16691_b200.sharded import shard_range, gather_rows
        squares = {}
        for n in (4096, 8192, 12288, 16384):
            sh = shard_range(n, rank, world, granule=256)
            m = sh.size
            dsq = alcop.gemm_desc(m, n, n, 1, alcop.BF16, alcop.BF16, alcop.B_KN)
            descs[(m, n, n)] = dsq
            ssq = sched.get((m, n, n)) or alcop.choose_schedule(dsq)
            sched[(m, n, n)] = ssq
            A = (torch.rand((m, n), device=dev) - 0.5).to(torch.bfloat16)
            B = (torch.rand((n, n), device=dev) - 0.5).to(torch.bfloat16)
            C = torch.empty((m, n), device=dev, dtype=torch.bfloat16)
            barrier()
            ms = time_graph(lambda i: launch(A, B, C, ssq, (m, n, n)), iters=8 if n < 12288 else 4, warmup=3)
            tt = torch.tensor([ms], device=dev, dtype=torch.float64)
            if world > 1:
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            tf = 2.0 * n ** 3 / (float(tt.item()) * 1e-3) / 1e12
            row = {"tflops_aggregate": round(tf, 1), "frac_of_peak_per_gpu": round(tf / world / peaks["bf16_tflops"], 3),
                   "rows_per_gpu": m, "schedule": ssq.as_dict()}
            if world > 1 and n == 16384:
                for _ in range(2):
                    gather_rows(C, n, rank, world, granule=256)
                torch.cuda.synchronize()
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record()
                gather_rows(C, n, rank, world, granule=256)
                e1.record()
                torch.cuda.synchronize()
                row["allgather_ms"] = round(e0.elapsed_time(e1), 3)
            squares[str(n)] = row
            del A, B, C
            torch.cuda.empty_cache()
        extra["large_square_m_sharded"] = {"sharding": "M (256-row granules), B replicated", "sizes": squares}

    # ---- e2e through the host-buffer ABI entry point (alcop_gemm_host)
    host = []
    for name, M, N, K in gemms:
        A = (torch.rand((M, K)) * 2 - 1).to(torch.bfloat16).pin_memory()
        B = (torch.rand((K, N)) * 2 - 1).to(torch.bfloat16).pin_memory()
        C = torch.empty((M, N), dtype=torch.bfloat16).pin_memory()
        host.append((A, B, C))
    # one workspace per GEMM of the step: the stream-ordered host entry point
    # overlaps the H2D of GEMM k+1 with the D2H of GEMM k (two copy engines)
    wss = [torch.empty(lib.alcop_gemm_workspace_bytes(ctypes.byref(descs[(M, N, K)])), dtype=torch.uint8,
                       device=dev) for _, M, N, K in gemms]

    def e2e_step():
        for (name, M, N, K), (A, B, C), ws in zip(gemms, host, wss):
            rc = lib.alcop_gemm_host_async(ctypes.byref(descs[(M, N, K)]), ctypes.byref(sched[(M, N, K)]),
                                           ctypes.c_void_p(A.data_ptr()), ctypes.c_void_p(B.data_ptr()),
                                           ctypes.c_void_p(C.data_ptr()), ctypes.c_void_p(ws.data_ptr()), sp)
            if rc:
                raise alcop.AlcopError(rc, lib.alcop_last_error().decode())
        torch.cuda.synchronize()  # the step's C blocks are on the host

    e2e_steps = max(3, min(args.steps, 20))
    for _ in range(2):
        e2e_step()
    torch.cuda.synchronize()
    barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        e2e_step()
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    te = torch.tensor([e2e_s], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_val = world * flops * e2e_steps / float(te.item()) / 1e12
    h2d = sum((M * K + K * N) * 2 for _, M, N, K in gemms)
    d2h = sum(M * N * 2 for _, M, N, K in gemms)

    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu:
            rows = ref_sample_rows(3.0)
            dt, cflops, kind, cores = cpu_reference_step(rows)
            cpu = {"value": cflops / dt / 1e12, "unit": UNIT, "cores": cores, "kind": kind,
                   "sample": "%d concurrent processes, each a %dx%d output block (full K) of one of the %d "
                             "BERT-layer GEMMs (round-robin) through the reference interpreter (pipec::run, "
                             "transformed program); %.2f s wall" % (cores, rows, REF_SAMPLE_COLS, len(BERT_GEMMS),
                                                                    dt)}
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
                "data": "synthetic (uniform[-1,1) bf16; %d rotating input sets, %.0f MB > 2x L2)"
                        % (nsets, nsets * set_bytes / 1e6),
                "config": {"workload": "bert_base_layer_gemms" + ("" if args.unfused_qkv else "_fused_qkv"),
                           "M": 4096,
                           "launch": "CUDA graph per input set: %d alcop_gemm launches chained with PDL" % len(gemms),
                           "gemms": {n: [M, N, K] for n, M, N, K in gemms}, "b_layout": "KN (reference)",
                           "parallelism": "replicas" if world > 1 else "single",
                           "l2": "inputs rotated over copies > 2x L2",
                           "schedule": ("alcop_tune (model rank, top %d timed on this GPU)" % TUNE_BUDGET
                                        if args.schedule == "tune" else "alcop_choose_schedule (model pick)"),
                           "schedules": {"%dx%dx%d" % k: v.as_dict() for k, v in sched.items()}},
                "gpu_launches": len(gemms) * args.steps,
                "clocks": {**clk.summary(), "sm_mhz_in_kernel": kclk,
                           "note": "sm_mhz: NVML samples during the timed region; sm_mhz_in_kernel: clock64 over "
                                   "%globaltimer in CTA 0 of the step's last GEMM under back-to-back steps (the "
                                   "loaded clock; NVML does not show it)"},
                "roofline": roofline,
                "cpu_baseline": cpu,
                "e2e": {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                        "entry_point": "alcop_gemm_host_async per GEMM (pinned host buffers; A row blocks H2D, "
                                       "multiplied as they land, C blocks D2H on a second copy stream), host "
                                       "sync at the end of every step"},
                "per_gemm": {k: {"tflops": round(v["tflops"], 1), "ms": round(v["ms"], 4), "shape": v["shape"],
                                 "frac_of_attainable": round(v["tflops"] / attainable(
                                     2.0 * v["shape"][0] * v["shape"][1] * v["shape"][2],
                                     2 * (v["shape"][0] * v["shape"][2] + v["shape"][2] * v["shape"][1]
                                          + v["shape"][0] * v["shape"][1])), 3),
                                 "launches_per_step": count[k]} for k, v in per.items()},
                ("step_fused_qkv" if args.unfused_qkv else "step_unfused_qkv"): alt,
                "step_one_launch": {"entry_point": "alcop_gemm_chain", **chain} if chain else None,
                **extra}
        print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="alcop", choices=["alcop", "reference"])
    ap.add_argument("--quick", action="store_true", help="skip the n_stage sweep and the large square")
    ap.add_argument("--schedule", default="tune", choices=["tune", "model"],
                    help="tune: time the model's top schedules per shape (alcop_tune); model: its first pick")
    ap.add_argument("--unfused-qkv", action="store_true", help="Q, K, V as three GEMMs (six launches per step)")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference_arm(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        main_gpu(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
