"""Pins the oracle (the C / numpy restatement in oracle/) to the reference
itself: every check compares against fixtures produced by the reference's own
code (oracle/_ref/ref_driver built from /root/reference, see
oracle/gen_golden.py)."""
import math

import numpy as np
import pytest

from oracle import coracle
from oracle.splitmix import random_tensor, splitmix_draws
from tests import golden_util as G


@pytest.fixture(scope="module", autouse=True)
def _built():
    coracle.lib()


def test_splitmix_matches_reference():
    for seed, d in G.splitmix().items():
        raw = [int(x) for x in d["raw"]]
        assert [int(x) for x in splitmix_draws(int(seed), len(raw))] == raw
        assert random_tensor(len(raw), int(seed)).tolist() == d["range"]
        assert coracle.random_tensor(len(raw), int(seed)).tolist() == d["range"]


@pytest.mark.parametrize("case", G.gemm_cases(), ids=lambda c: c["name"])
def test_gemm_outputs_match_interpreter(case):
    """The interpreter's int64 C (run(), interp.hpp:440) equals the oracle's
    exact GEMM and its fp32-accumulate GEMM over bf16 inputs."""
    M, N, K, b = case["M"], case["N"], case["K"], case["batch"]
    A = random_tensor(b * M * K, case["seed"] + 0).reshape((b, M, K) if b > 1 else (M, K))
    B = random_tensor(b * K * N, case["seed"] + 1).reshape((b, K, N) if b > 1 else (K, N))
    ref = G.output_c(case["name"]).reshape(-1)
    exact = coracle.gemm_i64(A, B).reshape(-1)
    assert np.array_equal(exact, ref)
    if M * N * K * b <= 1 << 24:
        Ah = coracle.to_dtype(A.astype(np.float32), "bf16")
        Bh = coracle.to_dtype(B.astype(np.float32), "bf16")
        C32 = coracle.gemm(Ah, Bh, "bf16", "f32").reshape(-1)
        assert np.array_equal(C32.astype(np.int64), ref)


def _single_level(c):
    return c["tA"] == 0 and c["tB"] == 0


@pytest.mark.parametrize("case", G.gemm_cases(), ids=lambda c: c["name"])
def test_root_index_algebra(case):
    """shift_and_wrap_indices + inject_prologues of a root pipeline
    (pipeline_pass.hpp:501-509, 647-656) restated in oracle_root_schedule."""
    walk = G.walk(case["name"])
    tileK = case["K"] // case["ko"]
    E = case["ko"]
    for side, s in (("A", case["sA"]), ("B", case["sB"])):
        if s < 2:
            continue
        buf = side + "_shared"
        got = G.producer_copies(walk, buf, tileK, case["batch"] > 1)
        ps, pc, cs = coracle.root_schedule(E, s)
        assert got == list(zip(ps.tolist(), pc.tolist()))
        if _single_level(case):
            cons = G.consumer_slots(walk, buf)
            assert len(cons) == E * case["ki"]
            assert [c[2] for c in cons] == [cs[c[0]] for c in cons]


@pytest.mark.parametrize("case", [c for c in G.gemm_cases() if not _single_level(c)], ids=lambda c: c["name"])
def test_nested_index_algebra(case):
    """The fused two-level algebra g = v*F + u + t-1 (pipeline_pass.hpp:510-527,
    657-676) restated in oracle_nested_schedule."""
    walk = G.walk(case["name"])
    E, F = case["ko"], case["ki"]
    for side, s, t in (("A", case["sA"], case["tA"]), ("B", case["sB"], case["tB"])):
        dst, src, src_u, src_v, cons = coracle.nested_schedule(E, F, s, t)
        copies = [e for e in walk if e["op"] == "copy" and e["dst"] == side + "_reg"]
        assert len(copies) == len(dst)
        for e, d, sl, u in zip(copies, dst, src, src_u):
            assert e["dstIdx"][0] == d
            assert e["srcIdx"][0] == sl
            k = e["srcIdx"][2] if side == "A" else e["srcIdx"][1]
            assert k == u
        reads = [(e["env"]["ko"], e["env"]["ki"], o["idx"][0]) for e in walk if e["op"] == "read"
                 for o in e["operands"] if o["buf"] == side + "_reg"]
        assert [r[2] for r in reads] == cons.tolist()


@pytest.mark.parametrize("case", G.gemm_cases(), ids=lambda c: c["name"])
def test_plan_fields(case):
    """predicateWaits = ceil((t-1)/F) and drainPairs (pipeline_pass.hpp:313,
    324-347) — including the root's s-1-dmax that causes the two-level leak."""
    for info in G.plan(case["name"]):
        side = info["buffer"][0]
        s = case["s" + side]
        t = case["t" + side]
        F = case["ki"]
        if info["level"] == 1:
            assert info["predicateWaits"] == math.ceil((t - 1) / F)
            assert info["drainPairs"] == t - 1
        else:
            dmax = math.ceil((t - 1) / F) if (t >= 2 and info["buffer"].endswith("_shared")) else 0
            assert info["drainPairs"] == info["stages"] - 1 - dmax


@pytest.mark.parametrize("case", G.gemm_cases(), ids=lambda c: c["name"])
def test_sync_trace_counters(case):
    """The interpreter's TraceEvent stream (interp.hpp:375-418) for the whole
    multi-tile program equals the restated event order + counters."""
    ref = G.trace(case["name"])
    got = coracle.sync_trace(G.tiles_of(case), case["ko"], case["ki"], case["sA"], case["sB"], case["tA"],
                             case["tB"], leak_fix=False)
    assert len(got) >= len(ref)
    for r, g in zip(ref, got):
        for k in ("kind", "group", "acquired", "committed", "waited", "released", "inflight"):
            assert r[k] == g[k], (r, g)
    if "config1" not in case["name"]:
        assert len(got) == len(ref)


def test_two_level_leak_and_fix():
    """The reference leaks one outer group per tile in two-level pipelines
    (SURVEY §0); the restated fix balances every group at the end."""
    leaky = coracle.sync_trace(4, 4, 4, 3, 3, 2, 2, leak_fix=False)
    fixed = coracle.sync_trace(4, 4, 4, 3, 3, 2, 2, leak_fix=True)

    def final(tr, grp):
        ev = [e for e in tr if e["group"] == grp]
        return ev[-1]

    assert final(leaky, "A_shared")["inflight"] == 4  # one leaked group per tile
    for grp in ("A_shared", "B_shared", "A_reg", "B_reg"):
        assert final(fixed, grp)["inflight"] == 0
    for e in fixed:
        assert e["released"] <= e["waited"] <= e["committed"] <= e["acquired"]


def _close(a, b):
    return abs(a - b) <= 1e-9 * max(1.0, abs(a), abs(b))


def test_model_matches_reference():
    hw = coracle.hw_default()
    L = coracle.lib()
    n_pred = 0
    for item in G.model_queries():
        q = item["q"].split()
        a = item["a"]
        fn, args = q[0], q[1:]
        if fn == "pipeline_latency":
            got = L.oracle_pipeline_latency(float(args[0]), float(args[1]), int(args[2]), int(args[3]), int(args[4]))
            assert _close(got, float(a)), item
        elif fn == "smem_load_latency":
            h = coracle.hw_default()
            h.bwLLC, h.bwDRAM, h.latLLCRead, h.latDRAMRead = map(float, args[3:7])
            assert _close(L.oracle_smem_load_latency(int(args[0]), int(args[1]), int(args[2]), h), float(a))
        elif fn == "epilogue_latency":
            h = coracle.hw_default()
            h.bwDRAMWrite, h.latDRAMWrite = float(args[2]), float(args[3])
            assert _close(L.oracle_epilogue_latency(int(args[0]), int(args[1]), h), float(a))
        elif fn == "compute_latency":
            h = coracle.hw_default()
            h.throughputSM = float(args[1])
            assert _close(L.oracle_compute_latency(int(args[0]), h, int(args[2]), int(args[3])), float(a))
        elif fn == "predict":
            got = coracle.predict([int(x) for x in args], hw)
            if a == "error":
                assert got is None, item
            else:
                want = [float(x) for x in a.split()]
                assert got is not None, item
                for g, w in zip(got, want):
                    assert _close(g, w), (item, got)
                n_pred += 1
    assert n_pred > 20


def test_spec_examples():
    """SPEC.md:438-475 numeric examples, through the restatement."""
    L = coracle.lib()
    assert L.oracle_pipeline_latency(0, 10, 8, 2, 1) == 80
    assert L.oracle_pipeline_latency(10, 10, 8, 2, 1) == 80
    assert L.oracle_pipeline_latency(30, 10, 8, 2, 1) == 160
    h = coracle.hw_default()
    assert L.oracle_smem_load_latency(4096, 1 << 20, 108, h) == 16784
    h.latDRAMWrite = 500
    assert L.oracle_epilogue_latency(8192, 108, h) == 28148


def test_fp_conversions_roundtrip():
    x = np.array([0.0, -0.0, 1.0, -2.5, 65504.0, 1e-8, 3.14159, 1.0 + 2 ** -9, 1.0 + 3 * 2 ** -9], dtype=np.float32)
    import torch
    for dt, tdt in (("bf16", torch.bfloat16), ("f16", torch.float16)):
        ours = coracle.to_f32(coracle.to_dtype(x, dt), dt)
        want = torch.from_numpy(x).to(tdt).float().numpy()
        assert np.array_equal(ours, want), (dt, ours, want)


def test_conv_oracle_equals_gemm_for_1x1():
    """A 1x1 stride-1 conv is the GEMM the reference can lower."""
    rng = np.random.RandomState(0)
    x = rng.randint(-8, 9, size=(2, 5, 6, 16)).astype(np.float32)
    w = rng.randint(-8, 9, size=(8, 1, 1, 16)).astype(np.float32)
    xh, wh = coracle.to_dtype(x, "bf16"), coracle.to_dtype(w, "bf16")
    y = coracle.conv2d(xh, wh, (1, 1), (0, 0), "bf16", "f32")
    A = x.reshape(-1, 16).astype(np.int64)
    B = w.reshape(8, 16).T.astype(np.int64)
    assert np.array_equal(y.reshape(-1, 8).astype(np.int64), coracle.gemm_i64(A, B))


@pytest.mark.parametrize("case", G.preop_cases(), ids=lambda c: c["name"])
def test_preop_outputs_match_interpreter(case):
    """gemm_schedule(w, preOp=true): C = mma(S2, B) with S2 = ew(A) = 2A+1
    (interp.hpp:363, 367-369), inlined (mma_ewa) or materialised."""
    M, N, K, b = case["M"], case["N"], case["K"], case["batch"]
    A = random_tensor(b * M * K, case["seed"] + 0).reshape((b, M, K) if b > 1 else (M, K))
    B = random_tensor(b * K * N, case["seed"] + 1).reshape((b, K, N) if b > 1 else (K, N))
    assert np.array_equal(coracle.gemm_i64(2 * A + 1, B).reshape(-1), G.output_c(case["name"]).reshape(-1))
