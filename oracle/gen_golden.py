"""Generates tests/golden/ from the reference itself (oracle/_ref/ref_driver,
compiled from the read-only headers under /root/reference).

TEST INFRASTRUCTURE.  Run here (the container that has /root/reference):
    make -C oracle all && python oracle/gen_golden.py
The fixtures are committed; the GPU box never needs /root/reference.
"""
import json
import os
import shutil
import subprocess
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
DRIVER = os.path.join(HERE, "_ref", "ref_driver")
GOLD = os.path.join(ROOT, "tests", "golden")


def script_text(split, hints, reg=False):
    lines = ["cache_read A shared", "cache_read B shared"]
    if reg:
        lines += ["cache_read A_shared register", "cache_read B_shared register"]
    lines.append("tile C " + " ".join("%s=%d" % kv for kv in split))
    for buf, n in hints:
        lines.append("pipeline %s %d" % (buf, n))
    return "\n".join(lines) + "\n"


def preop_script(split, hints, inline=True, reg=False):
    """gemm_schedule(w, preOp=true): S2 = ew(A) feeds the mma (schedule.hpp:73-86)."""
    lines = ["cache_read S2 shared", "cache_read B shared"]
    if reg:
        lines += ["cache_read S2_shared register", "cache_read B_shared register"]
    lines.append("tile C " + " ".join("%s=%d" % kv for kv in split))
    for buf, n in hints:
        lines.append("pipeline %s %d" % (buf, n))
    if inline:
        lines.append("inline S2")
    return "\n".join(lines) + "\n"


def split_of(M, N, K, tm, tn, ko, ki):
    return [("i0", M // tm), ("i1", tm), ("j0", N // tn), ("j1", tn), ("ko", ko), ("ki", ki)]


# (name, M, N, K, batch, tileM, tileN, ko, ki, sA, sB, tA, tB, mode)
GEMM_CASES = [
    ("s8_22", 8, 8, 8, 1, 4, 4, 4, 2, 2, 2, 0, 0, "strict"),
    ("s8_33", 8, 8, 8, 1, 4, 4, 4, 2, 3, 3, 0, 0, "strict"),
    ("s8_44", 8, 8, 8, 1, 4, 4, 4, 2, 4, 4, 0, 0, "strict"),
    ("s8_30", 8, 8, 8, 1, 4, 4, 4, 2, 3, 0, 0, 0, "strict"),
    ("s8_02", 8, 8, 8, 1, 4, 4, 4, 2, 0, 2, 0, 0, "strict"),
    ("s8_24", 8, 8, 8, 1, 4, 4, 4, 2, 2, 4, 0, 0, "strict"),
    ("s8_wrapE", 8, 8, 8, 1, 4, 4, 2, 4, 4, 4, 0, 0, "strict"),  # E=2 < s-1: prologue wraps
    ("s16_22", 16, 16, 16, 1, 8, 8, 8, 2, 2, 2, 0, 0, "strict"),
    ("s16_33", 16, 16, 16, 1, 8, 8, 8, 2, 3, 3, 0, 0, "strict"),
    ("s16_52", 16, 16, 16, 1, 8, 8, 8, 2, 5, 2, 0, 0, "strict"),
    ("s16_b3", 16, 8, 16, 3, 8, 4, 4, 4, 3, 3, 0, 0, "strict"),
    ("s32_rect", 32, 16, 64, 1, 16, 8, 16, 4, 4, 3, 0, 0, "strict"),
    ("t16_1tile", 8, 8, 16, 1, 8, 8, 4, 4, 3, 3, 2, 2, "strict"),
    ("t16_32", 8, 8, 16, 1, 4, 8, 4, 4, 3, 3, 2, 2, "stale"),
    ("t16_33", 16, 16, 16, 1, 8, 8, 4, 4, 3, 3, 3, 3, "stale"),
    ("t16_22", 16, 16, 16, 1, 8, 8, 4, 4, 2, 2, 2, 2, "stale"),
    ("t32_43", 16, 16, 32, 1, 8, 8, 8, 4, 4, 4, 3, 3, "stale"),
    ("t16_84", 16, 16, 16, 1, 16, 16, 8, 2, 3, 3, 4, 4, "strict"),
    ("t_b2", 8, 8, 16, 2, 8, 8, 4, 4, 3, 3, 2, 2, "stale"),
    # BASELINE config 1 exactly: fp16 512^3, tile 128x128x32, 2 smem + 2 inner stages
    ("config1", 512, 512, 512, 1, 128, 128, 16, 32, 2, 2, 2, 2, "stale"),
]

# pre-op programs (name, M, N, K, batch, script, mode): inline case 2 (mma_ewa) and the
# un-inlined (materialised S2) form
PREOP_CASES = [
    ("p8_inline", 8, 8, 8, 1, None, "strict"),
    ("p16_inline_33", 16, 16, 16, 1, None, "strict"),
    ("p16_materialised", 16, 16, 16, 1, None, "strict"),
    ("p16_inline_b2", 16, 8, 16, 2, None, "strict"),
]

# schedule-surface cases: (name, M, N, K, batch, script)
SCRIPT_CASES = [
    ("ok_single", 64, 64, 64, 1, script_text(split_of(64, 64, 64, 32, 32, 4, 16), [("A_shared", 3), ("B_shared", 3)])),
    ("ok_two_level", 64, 64, 64, 1, script_text(split_of(64, 64, 64, 32, 32, 4, 16),
                                                [("A_shared", 3), ("B_shared", 3), ("A_reg", 2), ("B_reg", 2)],
                                                reg=True)),
    ("ok_unhinted", 64, 64, 64, 1, script_text(split_of(64, 64, 64, 32, 32, 4, 16), [])),
    ("ok_comments", 64, 64, 64, 1, "# comment\ncache_read A shared  # trailing\n\ncache_read B shared\n"
                                   "tile C i0=2 i1=32 j0=2 j1=32 ko=4 ki=16\npipeline A_shared 2\n"),
    ("ordering_violation", 64, 64, 64, 1, "cache_read A shared\npipeline A_shared 2\n"),
    ("not_async_producer", 64, 64, 64, 1, "tile C i0=2 i1=32 j0=2 j1=32 ko=4 ki=16\npipeline A 2\n"),
    ("bad_stages", 64, 64, 64, 1, script_text(split_of(64, 64, 64, 32, 32, 4, 16), [("A_shared", 1)])),
    ("non_divisible", 64, 64, 64, 1, "cache_read A shared\ntile C i0=3 i1=32 j0=2 j1=32 ko=4 ki=16\n"),
    ("three_splits", 64, 64, 64, 1, "tile C i0=2 i1=4 i2=8 j0=2 j1=32 ko=4 ki=16\n"),
    ("missing_dim", 64, 64, 64, 1, "tile C i0=2 i1=32 ko=4 ki=16\n"),
    ("bad_split_name", 64, 64, 64, 1, "tile C x0=2 i1=32 j0=2 j1=32 ko=4 ki=16\n"),
    ("unknown_primitive", 64, 64, 64, 1, "vectorize C\n"),
    ("bad_scope", 64, 64, 64, 1, "cache_read A local\n"),
    ("scope_not_below", 64, 64, 64, 1, "cache_read A register\ncache_read A_reg shared\n"),
    ("duplicate_buffer", 64, 64, 64, 1, "cache_read A shared\ncache_read A shared\n"),
    ("inline_missing", 64, 64, 64, 1, "inline S2\n"),
    ("tile_non_output", 64, 64, 64, 1, "tile A i0=2 i1=32 j0=2 j1=32 ko=4 ki=16\n"),
    ("lookahead_exceeds", 64, 64, 64, 1, script_text(split_of(64, 64, 64, 32, 32, 64, 1),
                                                     [("A_shared", 2), ("A_reg", 3)], reg=True)),
    ("unsupported_nesting", 64, 64, 64, 1, "cache_read A shared\ncache_read A_shared register\n"
                                           "tile C i0=2 i1=32 j0=2 j1=32 ko=64\npipeline A_shared 2\n"
                                           "pipeline A_reg 2\n"),
    ("batched_ok", 32, 32, 32, 4, script_text(split_of(32, 32, 32, 16, 16, 2, 16), [("A_shared", 2), ("B_shared", 2)])),
    ("syntax_pipeline", 64, 64, 64, 1, "pipeline A_shared\n"),
    ("bad_extent", 64, 64, 64, 1, "tile C i0=2 i1=32 j0=2 j1=32 ko=4 ki=x\n"),
    ("zero_split", 64, 64, 64, 1, "tile C i0=0 i1=32 j0=2 j1=32 ko=4 ki=16\n"),
    ("one_level_k", 64, 64, 64, 1, "cache_read A shared\ncache_read B shared\ntile C i0=2 i1=32 j0=2 j1=32 ko=8\n"
                                   "pipeline A_shared 4\npipeline B_shared 2\n"),
    ("reg_only_hint", 64, 64, 64, 1, script_text(split_of(64, 64, 64, 32, 32, 4, 16), [("A_reg", 2)], reg=True)),
]
# (name, M, N, K, batch, script) with gemm_schedule(w, preOp=true)
PREOP_SCRIPT_CASES = [
    ("pre_inline_after_pipeline", 64, 64, 64, 1,
     preop_script(split_of(64, 64, 64, 32, 32, 4, 16), [("S2_shared", 3), ("B_shared", 3)])),
    ("pre_inline_before_pipeline", 64, 64, 64, 1,
     "cache_read S2 shared\ncache_read B shared\ntile C i0=2 i1=32 j0=2 j1=32 ko=4 ki=16\ninline S2\n"
     "pipeline S2_shared 2\n"),
    ("pre_materialised", 64, 64, 64, 1,
     preop_script(split_of(64, 64, 64, 32, 32, 4, 16), [("S2_shared", 2), ("B_shared", 2)], inline=False)),
    ("pre_inline_twice", 64, 64, 64, 1,
     preop_script(split_of(64, 64, 64, 32, 32, 4, 16), [("S2_shared", 2)]) + "inline S2\n"),
    ("pre_inline_no_consumer", 64, 64, 64, 1, "tile C i0=2 i1=32 j0=2 j1=32 ko=4 ki=16\ninline S2\n"),
    ("pre_inline_binary", 64, 64, 64, 1, "inline C\n"),
    ("pre_two_level", 64, 64, 64, 1,
     preop_script(split_of(64, 64, 64, 32, 32, 4, 16), [("S2_shared", 3), ("B_shared", 3), ("S2_reg", 2),
                                                         ("B_reg", 2)], reg=True)),
]

# model queries (SPEC.md:438-475 examples, then a deterministic grid)
MODEL_QUERIES = [
    "pipeline_latency 0 10 8 2 1", "pipeline_latency 10 10 8 2 1", "pipeline_latency 30 10 8 2 1",
    "smem_load_latency 4096 1048576 108 512 64 200 400", "epilogue_latency 8192 108 32 500",
    "compute_latency 16384 1024 4 2", "sim 0 10 8 1 1", "sim 30 10 64 2 1", "sim 10 10 64 4 1",
]


def model_grid():
    rng = np.random.RandomState(1234)
    qs = []
    for _ in range(400):
        M = int(rng.choice([512, 1024, 4096]))
        N = int(rng.choice([256, 768, 1024, 3072]))
        K = int(rng.choice([256, 768, 3072]))
        tM = int(rng.choice([32, 64, 128, 256]))
        tN = int(rng.choice([32, 64, 128, 256]))
        tK = int(rng.choice([8, 16, 32, 64]))
        rM = int(rng.choice([16, 32, 64]))
        rN = int(rng.choice([16, 32, 64]))
        rK = int(rng.choice([4, 8, 16]))
        sS = int(rng.randint(2, 6))
        sR = int(rng.randint(2, 4))
        nW = int(rng.choice([1, 2, 4, 8, 16]))
        qs.append("predict %d %d %d 1 %d %d %d %d %d %d %d %d %d" % (M, N, K, tM, tN, tK, rM, rN, rK, sS, sR, nW))
    for _ in range(100):
        qs.append("pipeline_latency %g %g %d %d %d" % (rng.randint(0, 500), rng.randint(1, 200), rng.randint(1, 64),
                                                       rng.randint(1, 8), rng.randint(1, 8)))
    return qs


def sim_grid():
    """pipe_sim.hpp:50-167: simulate_pipeline stats + traces and
    simulate_two_level (fused and restart) on a deterministic grid, incl. the
    ConfigError cases (counts < 1, negative times)."""
    rng = np.random.RandomState(4321)
    qs = ["sim 0 1 1 1 1", "sim 5 0 3 1 2", "sim 0 10 0 1 1", "sim -1 10 4 2 1", "sim 10 10 4 0 1",
          "simtrace 30 10 6 2 1", "simtrace 10 10 5 2 3", "simtrace 0 4 4 1 2",
          "sim2 100 10 8 2 5 10 4 2 1", "sim2 100 10 8 2 5 10 4 2 0", "sim2 0 10 0 2 5 10 4 2 1"]
    for _ in range(150):
        qs.append("sim %g %g %d %d %d" % (rng.randint(0, 400), rng.randint(0, 120), rng.randint(1, 40),
                                          rng.randint(1, 7), rng.randint(1, 5)))
    for _ in range(40):
        qs.append("simtrace %g %g %d %d %d" % (rng.randint(0, 100), rng.randint(1, 50), rng.randint(1, 8),
                                               rng.randint(1, 4), rng.randint(1, 4)))
    for _ in range(150):
        qs.append("sim2 %g %g %d %d %g %g %d %d %d" % (rng.randint(0, 2000), rng.randint(0, 50), rng.randint(1, 16),
                                                       rng.randint(1, 6), rng.randint(0, 100), rng.randint(1, 60),
                                                       rng.randint(1, 8), rng.randint(1, 4), rng.randint(0, 2)))
    return qs


def run(args, **kw):
    return subprocess.run([DRIVER] + args, check=True, capture_output=True, text=True, **kw)


def gen_gemm(outdir):
    os.makedirs(outdir, exist_ok=True)
    index = []
    for (name, M, N, K, batch, tm, tn, ko, ki, sA, sB, tA, tB, mode) in GEMM_CASES:
        reg = tA > 0 or tB > 0
        hints = []
        if sA:
            hints.append(("A_shared", sA))
        if sB:
            hints.append(("B_shared", sB))
        if tA:
            hints.append(("A_reg", tA))
        if tB:
            hints.append(("B_reg", tB))
        text = script_text(split_of(M, N, K, tm, tn, ko, ki), hints, reg)
        d = os.path.join(outdir, name)
        os.makedirs(d, exist_ok=True)
        with open(os.path.join(d, "script.txt"), "w") as f:
            f.write(text)
        with tempfile.TemporaryDirectory() as tmp:
            run(["gemm", "--M", str(M), "--N", str(N), "--K", str(K), "--batch", str(batch), "--script",
                 os.path.join(d, "script.txt"), "--outdir", tmp, "--mode", mode, "--seed", "0"])
            for f in ("plan.json", "run.json", "lowered.ir", "transformed.ir", "warnings.json"):
                shutil.copy(os.path.join(tmp, f), os.path.join(d, f))
            big = M * N * K * batch > 1 << 20
            if not big:
                shutil.copy(os.path.join(tmp, "walk.jsonl"), os.path.join(d, "walk.jsonl"))
                shutil.copy(os.path.join(tmp, "trace.jsonl"), os.path.join(d, "trace.jsonl"))
            else:
                # keep the first tile of the walk and a trace prefix
                with open(os.path.join(tmp, "walk.jsonl")) as f:
                    walk = [json.loads(l) for l in f]
                first = [w for w in walk if all(w["env"].get(v, 0) == 0 for v in ("i0", "j0", "b"))]
                with open(os.path.join(d, "walk.jsonl"), "w") as f:
                    for w in first:
                        f.write(json.dumps(w) + "\n")
                with open(os.path.join(tmp, "trace.jsonl")) as f, open(os.path.join(d, "trace.jsonl"), "w") as g:
                    for i, line in enumerate(f):
                        if i >= 4000:
                            break
                        g.write(line)
            C = np.fromfile(os.path.join(tmp, "C.bin"), dtype=np.int64)
            np.savez_compressed(os.path.join(d, "C.npz"), C=C.astype(np.int32))
        index.append({"name": name, "M": M, "N": N, "K": K, "batch": batch, "tileM": tm, "tileN": tn, "ko": ko,
                      "ki": ki, "sA": sA, "sB": sB, "tA": tA, "tB": tB, "mode": mode, "seed": 0})
        print("gemm", name, file=sys.stderr)
    with open(os.path.join(outdir, "index.json"), "w") as f:
        json.dump(index, f, indent=1)
    pre = []
    gen_preop(outdir, pre)
    with open(os.path.join(outdir, "preop_index.json"), "w") as f:
        json.dump(pre, f, indent=1)


def _preop_text(name, M, N, K):
    if name == "p8_inline":
        return preop_script(split_of(M, N, K, 4, 4, 4, 2), [("S2_shared", 2), ("B_shared", 2)])
    if name == "p16_inline_33":
        return preop_script(split_of(M, N, K, 8, 8, 8, 2), [("S2_shared", 3), ("B_shared", 3)])
    if name == "p16_materialised":
        return preop_script(split_of(M, N, K, 8, 8, 8, 2), [("S2_shared", 3), ("B_shared", 3)], inline=False)
    return preop_script(split_of(M, N, K, 8, 4, 4, 4), [("S2_shared", 2), ("B_shared", 2)])


def gen_preop(outdir, index):
    for (name, M, N, K, batch, _, mode) in PREOP_CASES:
        text = _preop_text(name, M, N, K)
        d = os.path.join(outdir, name)
        os.makedirs(d, exist_ok=True)
        with open(os.path.join(d, "script.txt"), "w") as f:
            f.write(text)
        with tempfile.TemporaryDirectory() as tmp:
            run(["gemm", "--M", str(M), "--N", str(N), "--K", str(K), "--batch", str(batch), "--script",
                 os.path.join(d, "script.txt"), "--outdir", tmp, "--mode", mode, "--seed", "0", "--preop", "1"])
            for f in ("plan.json", "run.json", "lowered.ir", "transformed.ir", "warnings.json", "walk.jsonl",
                      "trace.jsonl"):
                shutil.copy(os.path.join(tmp, f), os.path.join(d, f))
            C = np.fromfile(os.path.join(tmp, "C.bin"), dtype=np.int64)
            np.savez_compressed(os.path.join(d, "C.npz"), C=C.astype(np.int32))
        index.append({"name": name, "M": M, "N": N, "K": K, "batch": batch, "preop": 1, "mode": mode, "seed": 0})


def gen_scripts(path):
    out = []
    with tempfile.TemporaryDirectory() as tmp:
        for (name, M, N, K, batch, text) in SCRIPT_CASES:
            p = os.path.join(tmp, name + ".txt")
            with open(p, "w") as f:
                f.write(text)
            r = run(["script", "--M", str(M), "--N", str(N), "--K", str(K), "--batch", str(batch), "--script", p])
            res = json.loads(r.stdout)
            out.append({"name": name, "M": M, "N": N, "K": K, "batch": batch, "script": text, "result": res})
        for (name, M, N, K, batch, text) in PREOP_SCRIPT_CASES:
            p = os.path.join(tmp, name + ".txt")
            with open(p, "w") as f:
                f.write(text)
            r = run(["script", "--M", str(M), "--N", str(N), "--K", str(K), "--batch", str(batch), "--script", p,
                     "--preop", "1"])
            res = json.loads(r.stdout)
            out.append({"name": name, "M": M, "N": N, "K": K, "batch": batch, "script": text, "result": res,
                        "preop": 1})
    with open(path, "w") as f:
        for o in out:
            f.write(json.dumps(o) + "\n")


def gen_model(path):
    qs = MODEL_QUERIES + model_grid() + sim_grid()
    with tempfile.NamedTemporaryFile("w", suffix=".txt", delete=False) as f:
        f.write("\n".join(qs) + "\n")
        qpath = f.name
    r = run(["model", "--queries", qpath])
    os.unlink(qpath)
    res = r.stdout.strip().split("\n")
    assert len(res) == len(qs), (len(res), len(qs))
    with open(path, "w") as f:
        for q, a in zip(qs, res):
            f.write(json.dumps({"q": q, "a": a}) + "\n")


def gen_splitmix(path):
    out = {}
    for seed in (0, 1, 7, 1000003, 18446744073709551615):
        r = run(["splitmix", "--seed", str(seed), "--count", "64"])
        out[str(seed)] = json.loads(r.stdout)
    with open(path, "w") as f:
        json.dump(out, f)


def main():
    if not os.path.exists(DRIVER):
        raise SystemExit("build the reference driver first: make -C oracle ref")
    os.makedirs(GOLD, exist_ok=True)
    gen_splitmix(os.path.join(GOLD, "splitmix.json"))
    gen_model(os.path.join(GOLD, "model.jsonl"))
    gen_scripts(os.path.join(GOLD, "scripts.jsonl"))
    gen_gemm(os.path.join(GOLD, "gemm"))
    print("golden fixtures written to", GOLD)


if __name__ == "__main__":
    main()
