"""ctypes binding of oracle/liboracle.so (the C restatement).

TEST INFRASTRUCTURE: imported only by tests/, __graft_entry__.smoke() and
bench.py's CPU legs, always as the checker.
"""
import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "liboracle.so")
_lib = None


class OracleHW(ctypes.Structure):
    _fields_ = [("numSM", ctypes.c_int), ("throughputSM", ctypes.c_double), ("bwLLC", ctypes.c_double),
                ("bwDRAM", ctypes.c_double), ("bwDRAMWrite", ctypes.c_double), ("latLLCRead", ctypes.c_double),
                ("latDRAMRead", ctypes.c_double), ("latDRAMWrite", ctypes.c_double), ("bwSmem", ctypes.c_double),
                ("latSmem", ctypes.c_double), ("smemPerSM", ctypes.c_int64), ("regsPerSM", ctypes.c_int64),
                ("maxThreadblkPerSM", ctypes.c_int), ("maxWarpsPerSM", ctypes.c_int),
                ("utilKneeWarps", ctypes.c_int)]


def build():
    subprocess.run(["make", "-s", "-C", HERE, "oracle"], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build()
        L = ctypes.CDLL(LIB)
        i64, vp, dbl = ctypes.c_int64, ctypes.c_void_p, ctypes.c_double
        L.oracle_random_tensor.argtypes = [i64, ctypes.c_uint64, i64, i64, vp]
        L.oracle_convert.argtypes = [vp, ctypes.c_int, vp, ctypes.c_int, i64]
        L.oracle_gemm.argtypes = [i64, i64, i64, i64, vp, vp, vp, ctypes.c_int, ctypes.c_int, ctypes.c_int]
        L.oracle_gemm_i64.argtypes = [i64, i64, i64, i64, vp, vp, vp]
        L.oracle_conv2d.argtypes = [i64] * 7 + [ctypes.c_int] * 4 + [vp, vp, vp, ctypes.c_int, ctypes.c_int]
        L.oracle_random_i8.argtypes = [i64, ctypes.c_uint64, i64, i64, vp]
        L.oracle_gemm_rows_i8.argtypes = [i64, i64, i64, i64, vp, vp, ctypes.c_int, i64, vp, vp]
        L.oracle_gemm_cols_i8.argtypes = [i64, i64, i64, i64, vp, vp, ctypes.c_int, i64, vp, vp]
        L.oracle_conv2d_points_i8.argtypes = [i64] * 7 + [ctypes.c_int] * 4 + [vp, vp, i64, vp, vp]
        L.oracle_root_schedule.argtypes = [i64, i64, vp, vp, vp]
        L.oracle_nested_schedule.argtypes = [i64, i64, i64, i64, vp, vp, vp, vp, vp]
        L.oracle_sync_trace.argtypes = [i64, i64, i64, i64, i64, i64, i64, ctypes.c_int, vp, i64]
        L.oracle_sync_trace.restype = i64
        L.oracle_hw_default.argtypes = [ctypes.POINTER(OracleHW)]
        L.oracle_pipeline_latency.argtypes = [dbl, dbl, i64, ctypes.c_int, ctypes.c_int]
        L.oracle_pipeline_latency.restype = dbl
        L.oracle_smem_load_latency.argtypes = [i64, i64, i64, ctypes.POINTER(OracleHW)]
        L.oracle_smem_load_latency.restype = dbl
        L.oracle_epilogue_latency.argtypes = [i64, i64, ctypes.POINTER(OracleHW)]
        L.oracle_epilogue_latency.restype = dbl
        L.oracle_compute_latency.argtypes = [i64, ctypes.POINTER(OracleHW), ctypes.c_int, i64]
        L.oracle_compute_latency.restype = dbl
        L.oracle_predict.argtypes = [vp, ctypes.POINTER(OracleHW), vp]
        _lib = L
    return _lib


def _p(a):
    return ctypes.c_void_p(a.ctypes.data)


DT = {"f16": 0, "bf16": 1, "f32": 2}
NP = {"f16": np.uint16, "bf16": np.uint16, "f32": np.float32}


def random_tensor(count, seed, lo=-8, hi=8):
    out = np.empty(count, dtype=np.int64)
    lib().oracle_random_tensor(count, seed, lo, hi, _p(out))
    return out


def to_dtype(x_f32, dt):
    """fp32 array -> storage of dtype dt (RNE), as uint16 bits or float32."""
    x = np.ascontiguousarray(x_f32, dtype=np.float32)
    out = np.empty(x.shape, dtype=NP[dt])
    lib().oracle_convert(_p(x), 2, _p(out), DT[dt], x.size)
    return out


def to_f32(x, dt):
    x = np.ascontiguousarray(x)
    out = np.empty(x.shape, dtype=np.float32)
    lib().oracle_convert(_p(x), DT[dt], _p(out), 2, x.size)
    return out


def gemm(A, B, in_dt, out_dt, b_layout=0):
    """CPU fp32-accumulate GEMM/BMM on dtype storage arrays (see alcop_oracle.c §3)."""
    A = np.ascontiguousarray(A)
    B = np.ascontiguousarray(B)
    batched = A.ndim == 3
    batch = A.shape[0] if batched else 1
    M, K = A.shape[-2:]
    N = B.shape[-1] if b_layout == 0 else B.shape[-2]
    C = np.empty(((batch,) if batched else ()) + (M, N), dtype=NP[out_dt])
    lib().oracle_gemm(M, N, K, batch, _p(A), _p(B), _p(C), DT[in_dt], DT[out_dt], b_layout)
    return C


def gemm_i64(A, B):
    A = np.ascontiguousarray(A, dtype=np.int64)
    B = np.ascontiguousarray(B, dtype=np.int64)
    batched = A.ndim == 3
    batch = A.shape[0] if batched else 1
    M, K = A.shape[-2:]
    N = B.shape[-1]
    C = np.empty(((batch,) if batched else ()) + (M, N), dtype=np.int64)
    lib().oracle_gemm_i64(M, N, K, batch, _p(A), _p(B), _p(C))
    return C


def conv2d(x, w, stride, pad, in_dt, out_dt):
    x = np.ascontiguousarray(x)
    w = np.ascontiguousarray(w)
    N, H, W, C = x.shape
    K, R, S, _ = w.shape
    P = (H + 2 * pad[0] - R) // stride[0] + 1
    Q = (W + 2 * pad[1] - S) // stride[1] + 1
    y = np.empty((N, P, Q, K), dtype=NP[out_dt])
    lib().oracle_conv2d(N, H, W, C, K, R, S, stride[0], stride[1], pad[0], pad[1], _p(x), _p(w), _p(y),
                        DT[in_dt], DT[out_dt])
    return y


def random_i8(count, seed, lo=-8, hi=8):
    """random_tensor's draws (cli.hpp:41-46) as int8, element-parallel."""
    out = np.empty(count, dtype=np.int8)
    lib().oracle_random_i8(count, seed, lo, hi, _p(out))
    return out


def _bshape(A, B, b_layout):
    batched = A.ndim == 3
    batch = A.shape[0] if batched else 1
    M, K = A.shape[-2:]
    N = B.shape[-1] if b_layout == 0 else B.shape[-2]
    return M, N, K, batch


def gemm_rows_i8(A, B, rows, b_layout=0):
    """Exact rows (global index b*M + m) of A @ B on int8 D-int inputs -> int64 [len(rows), N]."""
    A = np.ascontiguousarray(A, dtype=np.int8)
    B = np.ascontiguousarray(B, dtype=np.int8)
    M, N, K, batch = _bshape(A, B, b_layout)
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    out = np.empty((len(rows), N), dtype=np.int64)
    lib().oracle_gemm_rows_i8(M, N, K, batch, _p(A), _p(B), b_layout, len(rows), _p(rows), _p(out))
    return out


def gemm_cols_i8(A, B, cols, b_layout=0):
    """Exact columns of A @ B for every (batch, row) -> int64 [batch*M, len(cols)]."""
    A = np.ascontiguousarray(A, dtype=np.int8)
    B = np.ascontiguousarray(B, dtype=np.int8)
    M, N, K, batch = _bshape(A, B, b_layout)
    cols = np.ascontiguousarray(cols, dtype=np.int64)
    out = np.empty((batch * M, len(cols)), dtype=np.int64)
    lib().oracle_gemm_cols_i8(M, N, K, batch, _p(A), _p(B), b_layout, len(cols), _p(cols), _p(out))
    return out


def conv2d_points_i8(x, w, stride, pad, pts):
    """Exact direct conv at output pixels pts [(n, p, q)] -> int64 [len(pts), K]."""
    x = np.ascontiguousarray(x, dtype=np.int8)
    w = np.ascontiguousarray(w, dtype=np.int8)
    N, H, W, C = x.shape
    K, R, S, _ = w.shape
    pts = np.ascontiguousarray(pts, dtype=np.int64).reshape(-1, 3)
    out = np.empty((len(pts), K), dtype=np.int64)
    lib().oracle_conv2d_points_i8(N, H, W, C, K, R, S, stride[0], stride[1], pad[0], pad[1], _p(x), _p(w),
                                  len(pts), _p(pts), _p(out))
    return out


def root_schedule(E, s):
    ps = np.empty(s - 1 + E, dtype=np.int64)
    pc = np.empty(s - 1 + E, dtype=np.int64)
    cs = np.empty(E, dtype=np.int64)
    lib().oracle_root_schedule(E, s, _p(ps), _p(pc), _p(cs))
    return ps, pc, cs


def nested_schedule(E, F, s, t):
    n = t - 1 + E * F
    arrs = [np.empty(n, dtype=np.int64) for _ in range(4)]
    cs = np.empty(E * F, dtype=np.int64)
    lib().oracle_nested_schedule(E, F, s, t, *[_p(a) for a in arrs], _p(cs))
    return arrs + [cs]


GROUPS = ["A_shared", "A_reg", "B_shared", "B_reg"]
KINDS = ["producer_acquire", "producer_commit", "consumer_wait", "consumer_release"]


def sync_trace(tiles, E, F, sA, sB, tA=0, tB=0, leak_fix=False):
    n = lib().oracle_sync_trace(tiles, E, F, sA, sB, tA, tB, int(leak_fix), None, 0)
    if n < 0:
        raise ValueError("shape not restated")
    out = np.zeros((max(n, 1), 7), dtype=np.int64)
    lib().oracle_sync_trace(tiles, E, F, sA, sB, tA, tB, int(leak_fix), _p(out), n)
    return [{"kind": KINDS[r[0]], "group": GROUPS[r[1]], "acquired": int(r[2]), "committed": int(r[3]),
             "waited": int(r[4]), "released": int(r[5]), "inflight": int(r[6])} for r in out[:n]]


def hw_default():
    h = OracleHW()
    lib().oracle_hw_default(ctypes.byref(h))
    return h


def predict(params, hw=None):
    p = np.array(params, dtype=np.int64)
    out = np.zeros(11, dtype=np.float64)
    rc = lib().oracle_predict(_p(p), ctypes.byref(hw or hw_default()), _p(out))
    return None if rc else out
