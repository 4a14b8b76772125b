"""paper_2210_16691_b200 — B200-native pipelined load-and-use GEMM / BMM /
implicit-GEMM conv (ALCOP, arXiv 2210.16691), behind the reference's schedule
surface.

The product is ``libalcop.so`` (C ABI in ``include/alcop.h``: sm_100a kernels +
C++ host code).  This module is a thin ctypes binding over that ABI so tests,
``bench.py`` and ``__graft_entry__`` can drive it with torch-allocated device
memory; it mirrors the reference's operator/schedule API names
(``gemm_schedule``/``apply_script``/``mark_pipeline`` hints,
``pipec::perf::predict``, ``tune::analytical_rank``) and its error classes.

There is no CPU fallback: every compute call goes through the CUDA kernels and
raises if the extension or a GPU is missing.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ALCOP_LIB", os.path.join(_HERE, "libalcop.so"))

ALCOP_OK = 0
ALCOP_ERR_PARSE = 2
ALCOP_ERR_VALIDATE = 3
ALCOP_ERR_ANALYSIS = 4
ALCOP_ERR_EQUIVALENCE = 5
ALCOP_ERR_CONFIG = 6
ALCOP_ERR_CUDA = 7

F16, BF16, F32 = 0, 1, 2
B_KN, B_NK = 0, 1
MODE_WRAP, MODE_FUSED = 0, 1

# every symbol include/alcop.h declares
EXPORTED_SYMBOLS = [
    "alcop_version", "alcop_last_error", "alcop_schedule_default", "alcop_parse_schedule_script",
    "alcop_validate", "alcop_smem_bytes", "alcop_enumerate_pipeline", "alcop_gemm", "alcop_gemm_traced",
    "alcop_gemm_workspace_bytes", "alcop_gemm_host", "alcop_gemm_host_async", "alcop_conv2d", "alcop_hw_default_b200",
    "alcop_hw_default_a100_reference", "alcop_predict", "alcop_choose_schedule", "alcop_ir_to_gemm",
    "alcop_tune", "alcop_simulate_pipeline", "alcop_simulate_two_level", "alcop_simulate_kernel",
    "alcop_gemm_chain_workspace_bytes", "alcop_gemm_chain", "alcop_shard_range", "alcop_gemm_sharded",
    "alcop_conv2d_sharded", "alcop_tune_workspace_bytes", "alcop_stream_k_workspace_bytes",
    "alcop_set_stream_k_workspace", "alcop_choose_conv_schedule",
]


class GemmDesc(ctypes.Structure):
    _fields_ = [("M", ctypes.c_int64), ("N", ctypes.c_int64), ("K", ctypes.c_int64), ("batch", ctypes.c_int64),
                ("in_dtype", ctypes.c_int32), ("out_dtype", ctypes.c_int32), ("b_layout", ctypes.c_int32),
                ("pre_op", ctypes.c_int32), ("lda", ctypes.c_int64), ("ldb", ctypes.c_int64),
                ("ldc", ctypes.c_int64), ("stride_a", ctypes.c_int64), ("stride_b", ctypes.c_int64),
                ("stride_c", ctypes.c_int64)]


CHAIN_MAX = 4


class Chain(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int32), ("dep", ctypes.c_int32 * CHAIN_MAX), ("desc", GemmDesc * CHAIN_MAX),
                ("A", ctypes.c_void_p * CHAIN_MAX), ("B", ctypes.c_void_p * CHAIN_MAX),
                ("C", ctypes.c_void_p * CHAIN_MAX)]


class Shard(ctypes.Structure):
    """alcop_shard: one shard of the multi-GPU driver (device, stream, operands)."""
    _fields_ = [("device", ctypes.c_int32), ("stream", ctypes.c_void_p), ("A", ctypes.c_void_p),
                ("B", ctypes.c_void_p), ("C", ctypes.c_void_p)]


class Schedule(ctypes.Structure):
    _fields_ = [("tileM", ctypes.c_int64), ("tileN", ctypes.c_int64), ("tileK", ctypes.c_int64),
                ("n_stage_smem_A", ctypes.c_int32), ("n_stage_smem_B", ctypes.c_int32),
                ("n_stage_inner", ctypes.c_int32), ("cta_group", ctypes.c_int32), ("mode", ctypes.c_int32),
                ("num_ctas", ctypes.c_int32), ("raster", ctypes.c_int32), ("stream_k", ctypes.c_int32)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_ if not f.startswith("reserved")}

    def __repr__(self):
        d = self.as_dict()
        return ("Schedule(tile=%dx%dx%d, stages A/B=%d/%d, inner=%d, mode=%s%s)"
                % (d["tileM"], d["tileN"], d["tileK"], d["n_stage_smem_A"], d["n_stage_smem_B"],
                   d["n_stage_inner"], "FUSED" if d["mode"] == MODE_FUSED else "WRAP",
                   (", cta_group=2" if d["cta_group"] == 2 else "") + (", stream_k" if d["stream_k"] else "")))


class ConvDesc(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int64) for n in ("N", "H", "W", "C", "K", "R", "S")] + \
               [(n, ctypes.c_int32) for n in ("stride_h", "stride_w", "pad_h", "pad_w", "in_dtype", "out_dtype",
                                               "x_halo", "reserved0")]


class HW(ctypes.Structure):
    _fields_ = [("numSM", ctypes.c_int32), ("throughputSM", ctypes.c_double), ("bwLLC", ctypes.c_double),
                ("bwDRAM", ctypes.c_double), ("bwDRAMWrite", ctypes.c_double), ("latLLCRead", ctypes.c_double),
                ("latDRAMRead", ctypes.c_double), ("latDRAMWrite", ctypes.c_double), ("bwSmem", ctypes.c_double),
                ("latSmem", ctypes.c_double), ("smemPerSM", ctypes.c_int64), ("regsPerSM", ctypes.c_int64),
                ("maxThreadblkPerSM", ctypes.c_int32), ("maxWarpsPerSM", ctypes.c_int32),
                ("utilKneeWarps", ctypes.c_int32), ("tmemColsPerSM", ctypes.c_int32), ("clockGHz", ctypes.c_double),
                ("tIssue", ctypes.c_double), ("tIssuePerBox", ctypes.c_double), ("tLaunch", ctypes.c_double),
                ("tTile", ctypes.c_double), ("overlapDRAM", ctypes.c_double), ("tPair", ctypes.c_double),
                ("tCapFlop", ctypes.c_double), ("tCapL2Byte", ctypes.c_double), ("tCapDramByte", ctypes.c_double),
                ("dramReusePair", ctypes.c_double), ("dramReusePairPerK", ctypes.c_double)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class Breakdown(ctypes.Structure):
    _fields_ = [(n, ctypes.c_double) for n in ("tKernel", "tThreadblk", "tInit", "tMainLoop", "tEpilogue",
                                                "tSmemLoad", "tRegLoad", "tSmemUse", "tCompute")] + \
               [(n, ctypes.c_int64) for n in ("nThreadblkBatch", "nThreadblkPerSM", "nThreadblkPerBatch",
                                               "nSmemLoop", "nRegLoop", "bytesOneSmemLoop", "bytesWorkset",
                                               "bytesOutputTile", "flopsOneRegLoop")] + \
               [(n, ctypes.c_double) for n in ("seconds", "bytesL2", "bytesDram", "tPower")]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class SimConfig(ctypes.Structure):
    _fields_ = [("tLoad", ctypes.c_double), ("tUse", ctypes.c_double), ("nLoop", ctypes.c_int64),
                ("nPipe", ctypes.c_int32), ("nMplx", ctypes.c_int32)]


class SimResult(ctypes.Structure):
    _fields_ = [(n, ctypes.c_double) for n in ("makespan", "firstComputeStart", "busy", "idleFraction",
                                                "comparable")]


class SimEvent(ctypes.Structure):
    _fields_ = [("time", ctypes.c_double), ("worker", ctypes.c_int32), ("kind", ctypes.c_int32),
                ("iteration", ctypes.c_int64)]


SIM_EVENT_NAMES = ("loadIssue", "loadDone", "computeStart", "computeEnd")  # pipe_sim.hpp:31-39


class SimKernel(ctypes.Structure):
    _fields_ = [(n, ctypes.c_double) for n in ("tKernel", "seconds", "tBody", "mmaBusy", "mmaIdleFraction",
                                                "tMainLoopTile", "tEpilogueTile", "tLoadChunk", "tUseChunk")] + \
               [("tilesPerUnit", ctypes.c_int64), ("loads", ctypes.c_int64)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class TuneTrial(ctypes.Structure):
    _fields_ = [("schedule", Schedule), ("predicted_s", ctypes.c_double), ("measured_s", ctypes.c_double)]


class Event(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in ("kind", "buf", "tile", "slot", "chunk", "parity", "acquired",
                                               "committed", "waited", "released")]


EVENT_FIELDS = [f for f, _ in Event._fields_]


class AlcopError(RuntimeError):
    """Raised on a non-zero ABI return; .code is the reference exit code, .rule the rule tag."""

    def __init__(self, code, message):
        self.code = code
        self.rule = message.split(":", 1)[0] if ":" in message else ""
        super().__init__("[%d] %s" % (code, message))


_lib = None


def load_library(path: str | None = None):
    """Loads libalcop.so; raises (no fallback) if it is missing."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = path or LIB_PATH
    if not os.path.exists(p):
        raise ImportError("libalcop.so not built (%s); run __graft_entry__.build()" % p)
    lib = ctypes.CDLL(p)
    P = ctypes.POINTER
    lib.alcop_version.restype = ctypes.c_char_p
    lib.alcop_last_error.restype = ctypes.c_char_p
    lib.alcop_schedule_default.argtypes = [P(Schedule)]
    lib.alcop_schedule_default.restype = None
    lib.alcop_parse_schedule_script.argtypes = [P(GemmDesc), ctypes.c_char_p, P(Schedule), ctypes.c_char_p,
                                                ctypes.c_size_t]
    lib.alcop_validate.argtypes = [P(GemmDesc), P(Schedule)]
    lib.alcop_smem_bytes.argtypes = [P(GemmDesc), P(Schedule)]
    lib.alcop_smem_bytes.restype = ctypes.c_int64
    lib.alcop_enumerate_pipeline.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32,
                                             ctypes.c_int32, ctypes.c_int32, P(Event), ctypes.c_int64,
                                             P(ctypes.c_int64)]
    lib.alcop_gemm.argtypes = [P(GemmDesc), P(Schedule), ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                               ctypes.c_void_p]
    lib.alcop_gemm_traced.argtypes = [P(GemmDesc), P(Schedule), ctypes.c_void_p, ctypes.c_void_p,
                                      ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p]
    lib.alcop_gemm_workspace_bytes.argtypes = [P(GemmDesc)]
    lib.alcop_gemm_workspace_bytes.restype = ctypes.c_int64
    lib.alcop_gemm_host.argtypes = [P(GemmDesc), P(Schedule), ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                    ctypes.c_void_p, ctypes.c_void_p]
    if hasattr(lib, "alcop_gemm_chain"):
        lib.alcop_gemm_chain_workspace_bytes.argtypes = [P(Chain)]
        lib.alcop_gemm_chain_workspace_bytes.restype = ctypes.c_int64
        lib.alcop_gemm_chain.argtypes = [P(Chain), P(Schedule), ctypes.c_void_p, ctypes.c_void_p]
    if hasattr(lib, "alcop_gemm_host_async"):
        lib.alcop_gemm_host_async.argtypes = lib.alcop_gemm_host.argtypes
    lib.alcop_conv2d.argtypes = [P(ConvDesc), P(Schedule), ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                 ctypes.c_void_p]
    lib.alcop_shard_range.argtypes = [ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, ctypes.c_int64,
                                      P(ctypes.c_int64), P(ctypes.c_int64)]
    lib.alcop_gemm_sharded.argtypes = [P(GemmDesc), P(Schedule), ctypes.c_int32, P(Shard), ctypes.c_int64]
    lib.alcop_conv2d_sharded.argtypes = [P(ConvDesc), P(Schedule), ctypes.c_int32, P(Shard)]
    lib.alcop_hw_default_b200.argtypes = [P(HW)]
    lib.alcop_hw_default_b200.restype = None
    lib.alcop_hw_default_a100_reference.argtypes = [P(HW)]
    lib.alcop_hw_default_a100_reference.restype = None
    lib.alcop_predict.argtypes = [P(GemmDesc), P(Schedule), P(HW), P(Breakdown)]
    lib.alcop_choose_schedule.argtypes = [P(GemmDesc), P(HW), P(Schedule)]
    lib.alcop_choose_conv_schedule.argtypes = [P(ConvDesc), P(HW), P(Schedule)]
    lib.alcop_ir_to_gemm.argtypes = [ctypes.c_char_p, P(GemmDesc), P(Schedule), ctypes.c_char_p, ctypes.c_size_t]
    lib.alcop_tune.argtypes = [P(GemmDesc), P(HW), ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                               ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, P(Schedule), P(TuneTrial),
                               ctypes.c_int32, P(ctypes.c_int32)]
    lib.alcop_tune_workspace_bytes.argtypes = [P(GemmDesc)]
    lib.alcop_tune_workspace_bytes.restype = ctypes.c_int64
    lib.alcop_stream_k_workspace_bytes.argtypes = [P(GemmDesc), P(Schedule)]
    lib.alcop_stream_k_workspace_bytes.restype = ctypes.c_int64
    lib.alcop_set_stream_k_workspace.argtypes = [ctypes.c_void_p, ctypes.c_int64]
    lib.alcop_simulate_pipeline.argtypes = [P(SimConfig), P(SimResult), P(SimEvent), ctypes.c_int64,
                                            P(ctypes.c_int64)]
    lib.alcop_simulate_two_level.argtypes = [P(SimConfig), P(SimConfig), ctypes.c_int32, P(ctypes.c_double)]
    lib.alcop_simulate_kernel.argtypes = [P(GemmDesc), P(Schedule), P(HW), P(SimKernel)]
    if path is None:
        _lib = lib
    return lib


def _check(rc):
    if rc != ALCOP_OK:
        raise AlcopError(rc, load_library().alcop_last_error().decode())


def version() -> str:
    return load_library().alcop_version().decode()


# ---------------------------------------------------------------- descriptors
_TORCH_DT = {}


def _dtype_code(dt) -> int:
    import torch
    m = {torch.float16: F16, torch.bfloat16: BF16, torch.float32: F32}
    if dt not in m:
        raise TypeError("unsupported dtype %s" % dt)
    return m[dt]


def gemm_desc(M, N, K, batch=1, in_dtype=BF16, out_dtype=BF16, b_layout=B_KN, **kw) -> GemmDesc:
    """WorkloadDesc (schedule.hpp:15-19) + the layouts lower() fixes (schedule.hpp:388-390)."""
    d = GemmDesc()
    d.M, d.N, d.K, d.batch = M, N, K, batch
    d.in_dtype, d.out_dtype, d.b_layout = in_dtype, out_dtype, b_layout
    for k, v in kw.items():
        setattr(d, k, v)
    return d


def default_schedule(**kw) -> Schedule:
    s = Schedule()
    load_library().alcop_schedule_default(ctypes.byref(s))
    for k, v in kw.items():
        setattr(s, k, v)
    return s


def make_schedule(tileN=256, tileK=64, n_stage=4, n_stage_inner=2, mode=MODE_FUSED, n_stage_B=None,
                  num_ctas=0, cta_group=1, raster=0, stream_k=0) -> Schedule:
    return default_schedule(tileM=128 * cta_group, tileN=tileN, tileK=tileK, n_stage_smem_A=n_stage,
                            n_stage_smem_B=n_stage if n_stage_B is None else n_stage_B,
                            n_stage_inner=n_stage_inner, mode=mode, num_ctas=num_ctas, cta_group=cta_group,
                            raster=raster, stream_k=stream_k)


def apply_script(desc: GemmDesc, script: str):
    """apply_script (schedule.hpp:590-646) on gemm_schedule(desc), mapped to a
    B200 Schedule.  Returns (schedule, warnings)."""
    s = Schedule()
    buf = ctypes.create_string_buffer(4096)
    _check(load_library().alcop_parse_schedule_script(ctypes.byref(desc), script.encode(), ctypes.byref(s), buf,
                                                      len(buf)))
    warns = [w for w in buf.value.decode().split("\n") if w]
    return s, warns


def validate(desc: GemmDesc, sched: Schedule):
    _check(load_library().alcop_validate(ctypes.byref(desc), ctypes.byref(sched)))


def smem_bytes(desc: GemmDesc, sched: Schedule) -> int:
    return load_library().alcop_smem_bytes(ctypes.byref(desc), ctypes.byref(sched))


def enumerate_pipeline(num_tiles, E, sA, sB, mode, role):
    """Host bookkeeping enumerator: list of event dicts for one CTA."""
    lib = load_library()
    n = ctypes.c_int64(0)
    _check(lib.alcop_enumerate_pipeline(num_tiles, E, sA, sB, mode, role, None, 0, ctypes.byref(n)))
    arr = (Event * max(1, n.value))()
    _check(lib.alcop_enumerate_pipeline(num_tiles, E, sA, sB, mode, role, arr, n.value, ctypes.byref(n)))
    return [{f: getattr(arr[i], f) for f in EVENT_FIELDS} for i in range(n.value)]


def hw_b200(burst: bool = False) -> HW:
    """B200 model constants.  Default: the sustained (power-capped) regime a
    long run of GEMMs is in; burst=True zeroes the power-cap terms (a kernel
    timed alone, in short bursts, at full clock)."""
    h = HW()
    load_library().alcop_hw_default_b200(ctypes.byref(h))
    if burst:
        h.tCapFlop = h.tCapL2Byte = h.tCapDramByte = 0.0
    return h


def hw_a100_reference() -> HW:
    h = HW()
    load_library().alcop_hw_default_a100_reference(ctypes.byref(h))
    return h


def predict(desc: GemmDesc, sched: Schedule, hw: HW | None = None) -> dict:
    b = Breakdown()
    _check(load_library().alcop_predict(ctypes.byref(desc), ctypes.byref(sched), ctypes.byref(hw or hw_b200()),
                                        ctypes.byref(b)))
    return b.as_dict()


def choose_schedule(desc: GemmDesc, hw: HW | None = None) -> Schedule:
    s = Schedule()
    _check(load_library().alcop_choose_schedule(ctypes.byref(desc), ctypes.byref(hw or hw_b200()),
                                                ctypes.byref(s)))
    return s


def sim_config(tLoad, tUse, nLoop, nPipe=1, nMplx=1) -> SimConfig:
    """SimConfig (pipe_sim.hpp:16-22)."""
    return SimConfig(float(tLoad), float(tUse), int(nLoop), int(nPipe), int(nMplx))


def simulate_pipeline(cfg: SimConfig, trace=False):
    """simulate_pipeline (pipe_sim.hpp:55-127): a dict of the SimResult
    fields (+ "comparable" = comparable_worker_latency); with trace=True also
    "trace": [(time, worker, kind_name, iteration)] sorted by time."""
    lib = load_library()
    r = SimResult()
    n = ctypes.c_int64(0)
    cap = 4 * cfg.nLoop * cfg.nMplx if trace and cfg.nLoop > 0 and cfg.nMplx > 0 else 0
    buf = (SimEvent * max(1, cap))() if trace else None
    _check(lib.alcop_simulate_pipeline(ctypes.byref(cfg), ctypes.byref(r), buf, cap,
                                       ctypes.byref(n) if trace else None))
    out = {f: getattr(r, f) for f, _ in r._fields_}
    if trace:
        out["trace"] = [(e.time, e.worker, SIM_EVENT_NAMES[e.kind], e.iteration) for e in buf[:n.value]]
    return out


def simulate_two_level(outer: SimConfig, inner: SimConfig, fused=True) -> float:
    """simulate_two_level (pipe_sim.hpp:138-167)."""
    m = ctypes.c_double(0)
    _check(load_library().alcop_simulate_two_level(ctypes.byref(outer), ctypes.byref(inner), 1 if fused else 0,
                                                   ctypes.byref(m)))
    return m.value


def simulate_kernel(desc: GemmDesc, sched: Schedule, hw: HW | None = None) -> dict:
    """B200 two-level kernel simulation: smem ring x TMEM accumulator ring per
    persistent CTA, with alcop_predict's chunk and epilogue times."""
    k = SimKernel()
    _check(load_library().alcop_simulate_kernel(ctypes.byref(desc), ctypes.byref(sched), ctypes.byref(hw or hw_b200()),
                                                ctypes.byref(k)))
    return k.as_dict()


# ---------------------------------------------------------------- compute
def _stream_ptr(stream=None):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _require_cuda(*ts):
    for t in ts:
        if not t.is_cuda:
            raise RuntimeError("alcop compute entry points take CUDA tensors (no CPU fallback)")


def _gemm_operands(A, B, b_layout, out=None, out_dtype=None):
    """Shape / dtype checks of a (batched) GEMM call before anything reaches
    the ABI: the descriptor is built from these shapes, so a mismatch would let
    the kernel read or write outside the buffers.  Returns (M, N, K, batch,
    batched, out_dtype)."""
    if A.dim() not in (2, 3) or B.dim() != A.dim():
        raise ValueError("matmul: A and B must both be 2-D or both 3-D (batched); got %d-D and %d-D"
                         % (A.dim(), B.dim()))
    if A.dtype != B.dtype:
        raise TypeError("matmul: A and B dtypes differ (%s, %s)" % (A.dtype, B.dtype))
    batched = A.dim() == 3
    M, K = A.shape[-2], A.shape[-1]
    if b_layout == B_KN:
        Kb, N = B.shape[-2], B.shape[-1]
    elif b_layout == B_NK:
        N, Kb = B.shape[-2], B.shape[-1]
    else:
        raise ValueError("matmul: b_layout must be B_KN or B_NK")
    if Kb != K:
        raise ValueError("matmul: reduction sizes differ (A has K=%d, B has K=%d)" % (K, Kb))
    batch = A.shape[0] if batched else 1
    if batched and B.shape[0] != batch:
        raise ValueError("matmul: batch sizes differ (%d, %d)" % (batch, B.shape[0]))
    out_dtype = out_dtype or (out.dtype if out is not None else A.dtype)
    if out is not None:
        want = ((batch,) if batched else ()) + (M, N)
        if tuple(out.shape) != want:
            raise ValueError("matmul: out has shape %s, expected %s" % (tuple(out.shape), want))
        if out.dtype != out_dtype:
            raise TypeError("matmul: out dtype %s != out_dtype %s" % (out.dtype, out_dtype))
        if not out.is_contiguous():
            raise ValueError("matmul: out must be contiguous")
        if out.device != A.device:
            raise ValueError("matmul: out is on %s, A on %s" % (out.device, A.device))
    return M, N, K, batch, batched, out_dtype


def matmul(A, B, sched: Schedule | None = None, out_dtype=None, b_layout=B_KN, out=None, stream=None, pre_op=0):
    """Pipelined matmul C = A @ B (or batched) through alcop_gemm; pre_op=1
    computes C = (2A+1) @ B with f fused into the pipeline (the reference's
    inlined elementwise pre-op).

    A: [M,K] or [b,M,K]; B: [K,N] / [b,K,N] (b_layout B_KN, the reference
    layout) or [N,K] / [b,N,K] (B_NK).  fp16/bf16 in, fp32 accumulate.
    Shapes, dtypes and `out` are checked (no broadcasting)."""
    import torch
    M, N, K, batch, batched, out_dtype = _gemm_operands(A, B, b_layout, out, out_dtype)
    _require_cuda(A, B)
    if out is None:
        out = torch.empty(((batch,) if batched else ()) + (M, N), dtype=out_dtype, device=A.device)
    A = A.contiguous()
    B = B.contiguous()
    d = gemm_desc(M, N, K, batch, _dtype_code(A.dtype), _dtype_code(out_dtype), b_layout, pre_op=pre_op)
    # the model ranks the space valid for this descriptor (with pre_op: the
    # single-CTA kernel with the transform warps and its shared-memory budget)
    s = sched if sched is not None else choose_schedule(d)
    _check(load_library().alcop_gemm(ctypes.byref(d), ctypes.byref(s), ctypes.c_void_p(A.data_ptr()),
                                     ctypes.c_void_p(B.data_ptr()), ctypes.c_void_p(out.data_ptr()),
                                     _stream_ptr(stream)))
    return out


def matmul_traced(A, B, sched: Schedule, out_dtype=None, b_layout=B_KN, events_cap=None):
    """matmul with the device debug trace; returns (C, trace[cta][role] -> list of event dicts)."""
    import torch
    M, N, K, batch, batched, out_dtype = _gemm_operands(A, B, b_layout, None, out_dtype)
    _require_cuda(A, B)
    A = A.contiguous()
    B = B.contiguous()
    out = torch.empty(((batch,) if batched else ()) + (M, N), dtype=out_dtype, device=A.device)
    d = gemm_desc(M, N, K, batch, _dtype_code(A.dtype), _dtype_code(out_dtype), b_layout)
    tiles = -(-M // 128) * -(-N // sched.tileN) * batch
    sms = torch.cuda.get_device_properties(A.device).multi_processor_count
    ctas = min(tiles, sched.num_ctas if sched.num_ctas > 0 else sms)
    E = -(-K // sched.tileK)
    per_cta = -(-tiles // ctas)
    cap = events_cap or (per_cta * (E + 32) * 4 + 64)
    tr = torch.full((ctas, 2, cap, len(EVENT_FIELDS)), -7, dtype=torch.int32, device=A.device)
    _check(load_library().alcop_gemm_traced(ctypes.byref(d), ctypes.byref(sched), ctypes.c_void_p(A.data_ptr()),
                                            ctypes.c_void_p(B.data_ptr()), ctypes.c_void_p(out.data_ptr()),
                                            ctypes.c_void_p(tr.data_ptr()), cap, _stream_ptr()))
    torch.cuda.synchronize()
    host = tr.cpu().numpy()
    traces = []
    for c in range(ctas):
        roles = []
        for r in range(2):
            rows = host[c, r]
            valid = rows[:, 0] != -7
            roles.append([dict(zip(EVENT_FIELDS, map(int, row))) for row in rows[valid]])
        traces.append(roles)
    return out, traces


def matmul_host(A_host, B_host, sched: Schedule, out_dtype, b_layout=B_KN, C_host=None, workspace=None,
                stream=None):
    """End-to-end call with HOST (pinned) tensors through alcop_gemm_host:
    H2D copies, kernel, D2H copy, synchronous.  Returns C_host."""
    import torch
    if A_host.is_cuda or B_host.is_cuda:
        raise ValueError("matmul_host takes host (pinned) tensors")
    if not (A_host.is_contiguous() and B_host.is_contiguous()):
        raise ValueError("matmul_host takes packed (contiguous) host tensors")
    M, N, K, batch, batched, out_dtype = _gemm_operands(A_host, B_host, b_layout, None, out_dtype)
    d = gemm_desc(M, N, K, batch, _dtype_code(A_host.dtype), _dtype_code(out_dtype), b_layout)
    if C_host is not None:
        want = ((batch,) if batched else ()) + (M, N)
        if tuple(C_host.shape) != want or C_host.dtype != out_dtype or not C_host.is_contiguous() or C_host.is_cuda:
            raise ValueError("matmul_host: C_host must be a contiguous host %s tensor of shape %s" % (out_dtype, want))
    if C_host is None:
        C_host = torch.empty(((batch,) if batched else ()) + (M, N), dtype=out_dtype, pin_memory=True)
    if workspace is None:
        workspace = torch.empty(load_library().alcop_gemm_workspace_bytes(ctypes.byref(d)), dtype=torch.uint8,
                                device="cuda")
    _check(load_library().alcop_gemm_host(ctypes.byref(d), ctypes.byref(sched),
                                          ctypes.c_void_p(A_host.data_ptr()), ctypes.c_void_p(B_host.data_ptr()),
                                          ctypes.c_void_p(C_host.data_ptr()), ctypes.c_void_p(workspace.data_ptr()),
                                          _stream_ptr(stream)))
    return C_host


def conv_desc(N, H, W, C, K, R, S, stride=(1, 1), pad=(0, 0), in_dtype=BF16, out_dtype=BF16) -> ConvDesc:
    d = ConvDesc()
    d.N, d.H, d.W, d.C, d.K, d.R, d.S = N, H, W, C, K, R, S
    d.stride_h, d.stride_w = stride
    d.pad_h, d.pad_w = pad
    d.in_dtype, d.out_dtype = in_dtype, out_dtype
    return d


def conv_out_hw(H, W, R, S, stride, pad):
    return (H + 2 * pad[0] - R) // stride[0] + 1, (W + 2 * pad[1] - S) // stride[1] + 1


def conv2d(x, w, stride=(1, 1), pad=(0, 0), sched: Schedule | None = None, out_dtype=None, out=None, stream=None,
           x_halo=False):
    """Implicit-GEMM conv2d through alcop_conv2d: x NHWC, w KRSC -> y NPQK
    (fp16/bf16 in, fp32 accumulate).  Default schedule: the model's pick for
    the GEMM view (M=N*P*Q, N=K, K=R*S*C) with tileK 64.  x_halo=True: x is
    stored with its zero padding halo, [N, H+2*pad_h, W+2*pad_w, C] (enables
    the one-box-per-filter-row kernel when S*C <= 64).  C <= 4 with
    horizontal stride 2 (ResNet-50 conv1) runs on the stem kernel
    (csrc/stem_sm100.cu) with the channels padded to 4; other C % 8 != 0
    are padded to 8."""
    import torch
    _require_cuda(x, w)
    ob = 4 if (out_dtype or (out.dtype if out is not None else x.dtype)) == torch.float32 else 2
    if (x.shape[-1] <= 4 and not x_halo and stride[1] == 2 and x.shape[2] % 16 == 0 and w.shape[0] % 16 == 0
            and w.shape[0] <= 256 and (w.shape[0] * ob) % 128 == 0):
        # the stem kernel: C = 4 (pixel pairs are 16-byte UMMA rows); zero channels contribute nothing
        if x.shape[-1] < 4:
            x = torch.nn.functional.pad(x, (0, 4 - x.shape[-1]))
            w = torch.nn.functional.pad(w, (0, 4 - w.shape[-1]))
    elif x.shape[-1] % 8:
        # NHWC channel padding to the 16-byte TMA granule (ResNet-50 conv1: 3 -> 8); zero filter
        # channels make the padded taps contribute nothing
        padc = 8 - x.shape[-1] % 8
        x = torch.nn.functional.pad(x, (0, padc))
        w = torch.nn.functional.pad(w, (0, padc))
    N, H, W, C = x.shape
    if x_halo:
        H, W = H - 2 * pad[0], W - 2 * pad[1]
    K, R, S, _ = w.shape
    P, Q = conv_out_hw(H, W, R, S, stride, pad)
    if w.dim() != 4 or w.shape[-1] != C or w.dtype != x.dtype:
        raise ValueError("conv2d: w must be KRSC with x's channel count and dtype (x %s %s, w %s %s)"
                         % (tuple(x.shape), x.dtype, tuple(w.shape), w.dtype))
    out_dtype = out_dtype or (out.dtype if out is not None else x.dtype)
    if out is None:
        out = torch.empty((N, P, Q, K), dtype=out_dtype, device=x.device)
    elif tuple(out.shape) != (N, P, Q, K) or out.dtype != out_dtype or not out.is_contiguous():
        raise ValueError("conv2d: out must be a contiguous %s tensor of shape %s" % (out_dtype, (N, P, Q, K)))
    d = conv_desc(N, H, W, C, K, R, S, stride, pad, _dtype_code(x.dtype), _dtype_code(out_dtype))
    d.x_halo = 1 if x_halo else 0
    if sched is None:
        sched = choose_conv_schedule(d)
    # keep the contiguous operands alive across the launch: a temporary freed
    # before the kernel runs could be reused by the other operand's copy
    xc = x.contiguous()
    wc = w.contiguous()
    if stream is not None:  # the launch stream is not the one the allocator ties the copies to
        xc.record_stream(stream)
        wc.record_stream(stream)
    _check(load_library().alcop_conv2d(ctypes.byref(d), ctypes.byref(sched), ctypes.c_void_p(xc.data_ptr()),
                                       ctypes.c_void_p(wc.data_ptr()), ctypes.c_void_p(out.data_ptr()),
                                       _stream_ptr(stream)))
    del xc, wc
    return out


def choose_conv_schedule(conv: ConvDesc, hw: HW | None = None) -> Schedule:
    """alcop_choose_conv_schedule: the model's pick over the conv kernel's space."""
    s = Schedule()
    _check(load_library().alcop_choose_conv_schedule(ctypes.byref(conv), ctypes.byref(hw or hw_b200()),
                                                     ctypes.byref(s)))
    return s


def ir_to_gemm(ir_text: str):
    """Reference IR (`pipec schedule` output) -> (GemmDesc, Schedule, info)."""
    d, s = GemmDesc(), Schedule()
    buf = ctypes.create_string_buffer(512)  # noqa
    _check(load_library().alcop_ir_to_gemm(ir_text.encode(), ctypes.byref(d), ctypes.byref(s), buf, len(buf)))
    return d, s, buf.value.decode()


def run_ir(ir_text: str, inputs: dict, stream=None):
    """The reference's `run` workflow on B200: inputs {"A": int/float array, "B": ...}
    laid out as the IR declares them; returns {"C": float32 array} (exact for the
    reference's integer inputs)."""
    import numpy as np
    import torch
    d, s, _ = ir_to_gemm(ir_text)
    A = torch.as_tensor(np.asarray(inputs["A"], dtype=np.float32)).to(torch.float16).cuda()
    B = torch.as_tensor(np.asarray(inputs["B"], dtype=np.float32)).to(torch.float16).cuda()
    shp = ((d.batch,) if d.batch > 1 else ()) + (d.M, d.N)
    C = torch.empty(shp, dtype=torch.float32, device="cuda")
    _check(load_library().alcop_gemm(ctypes.byref(d), ctypes.byref(s), ctypes.c_void_p(A.data_ptr()),
                                     ctypes.c_void_p(B.data_ptr()), ctypes.c_void_p(C.data_ptr()),
                                     _stream_ptr(stream)))
    torch.cuda.synchronize()
    return {"C": C.cpu().numpy()}


def tune(A, B, C, budget=8, b_layout=B_KN, hw: HW | None = None, stream=None):
    """Model-assisted tuning on the GPU (alcop_tune): rank the B200 space with
    the analytical model, time the top `budget` schedules on (A, B, C), return
    (best schedule, [trials in model rank order])."""
    batched = A.dim() == 3
    M, K = A.shape[-2], A.shape[-1]
    N = B.shape[-1] if b_layout == B_KN else B.shape[-2]
    d = gemm_desc(M, N, K, A.shape[0] if batched else 1, _dtype_code(A.dtype), _dtype_code(C.dtype), b_layout)
    import torch
    best = Schedule()
    cap = max(1, budget)
    arr = (TuneTrial * cap)()
    n = ctypes.c_int32(0)
    lib = load_library()
    wsb = lib.alcop_tune_workspace_bytes(ctypes.byref(d))
    ws = torch.empty(max(1, wsb), dtype=torch.uint8, device=A.device)  # caller-owned (the library never allocates)
    _check(lib.alcop_tune(ctypes.byref(d), ctypes.byref(hw or hw_b200()), budget, ctypes.c_void_p(A.data_ptr()),
                          ctypes.c_void_p(B.data_ptr()), ctypes.c_void_p(C.data_ptr()), ctypes.c_void_p(ws.data_ptr()),
                          wsb, _stream_ptr(stream), ctypes.byref(best), arr, cap, ctypes.byref(n)))
    del ws
    return best, [{"schedule": arr[i].schedule.as_dict(), "predicted_s": arr[i].predicted_s,
                   "measured_s": arr[i].measured_s} for i in range(n.value)]


def make_chain(gemms, dep=None, b_layout=B_KN) -> Chain:
    """gemms: [(A, B, C), ...] CUDA tensors (A [M,K], B [K,N] or [N,K], C [M,N]);
    dep[p] = 1: A_p row blocks wait for C_{p-1} row blocks (alcop_gemm_chain)."""
    ch = Chain()
    ch.n = len(gemms)
    for i, (A, B, C) in enumerate(gemms):
        M, K = A.shape
        N = B.shape[1] if b_layout == B_KN else B.shape[0]
        ch.desc[i] = gemm_desc(M, N, K, 1, _dtype_code(A.dtype), _dtype_code(C.dtype), b_layout)
        ch.A[i], ch.B[i], ch.C[i] = A.data_ptr(), B.data_ptr(), C.data_ptr()
        ch.dep[i] = int(dep[i]) if dep else 0
    return ch


def gemm_chain(gemms, sched: Schedule, dep=None, b_layout=B_KN, workspace=None, stream=None):
    """Several GEMMs in one persistent launch (alcop_gemm_chain); returns the Chain."""
    import torch
    ch = make_chain(gemms, dep, b_layout)
    lib = load_library()
    if workspace is None:
        workspace = torch.empty(max(4, lib.alcop_gemm_chain_workspace_bytes(ctypes.byref(ch))), dtype=torch.uint8,
                                device=gemms[0][0].device)
    _check(lib.alcop_gemm_chain(ctypes.byref(ch), ctypes.byref(sched), ctypes.c_void_p(workspace.data_ptr()),
                                _stream_ptr(stream)))
    return ch


# ---------------------------------------------------------------- multi-GPU driver (C ABI)
def shard_range(total, rank, world, granule=1):
    """alcop_shard_range: (start, count) of shard `rank`."""
    a, n = ctypes.c_int64(0), ctypes.c_int64(0)
    _check(load_library().alcop_shard_range(total, rank, world, granule, ctypes.byref(a), ctypes.byref(n)))
    return a.value, n.value


def gemm_sharded(desc: GemmDesc, shards, sched: Schedule | None = None, granule=256):
    """alcop_gemm_sharded: shards = [(device, stream, A_shard, B_replica, C_shard)] with torch CUDA tensors
    (A/C: this shard's rows, or batch entries when desc.batch > 1); one host thread per shard."""
    arr = (Shard * len(shards))()
    for i, (dev, st, A, B, C) in enumerate(shards):
        arr[i] = Shard(dev, st.cuda_stream if st is not None else None, A.data_ptr() if A is not None else None,
                       B.data_ptr() if B is not None else None, C.data_ptr() if C is not None else None)
    _check(load_library().alcop_gemm_sharded(ctypes.byref(desc), ctypes.byref(sched) if sched is not None else None,
                                             len(shards), arr, granule))


def conv2d_sharded(desc: ConvDesc, sched: Schedule, shards):
    """alcop_conv2d_sharded: shards = [(device, stream, x_images, w_replica, y_images)]."""
    arr = (Shard * len(shards))()
    for i, (dev, st, x, w, y) in enumerate(shards):
        arr[i] = Shard(dev, st.cuda_stream if st is not None else None, x.data_ptr() if x is not None else None,
                       w.data_ptr() if w is not None else None, y.data_ptr() if y is not None else None)
    _check(load_library().alcop_conv2d_sharded(ctypes.byref(desc), ctypes.byref(sched), len(shards), arr))


_SK_WS = {}


def set_stream_k_workspace(nbytes=64 << 20, device=None):
    """Registers a caller-owned stream-K workspace (fp32 partials + flags) for
    the current device (alcop_set_stream_k_workspace); kept alive here."""
    import torch
    dev = torch.device("cuda", device if device is not None else torch.cuda.current_device())
    ws = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    with torch.cuda.device(dev):
        _check(load_library().alcop_set_stream_k_workspace(ctypes.c_void_p(ws.data_ptr()), nbytes))
    _SK_WS[dev.index] = ws
    return ws
