"""Generates tests/golden/scripts_fuzz.jsonl: seeded random schedule scripts
run through the reference itself (oracle/_ref/ref_driver `script`:
apply_script(gemm_schedule(w, preOp)) -> lower -> analyze_pipelines ->
transform, schedule.hpp:73-646, pipeline_pass.hpp:184-764), recording the
accept/reject decision, the exception class and rule tag, and the plan.

TEST INFRASTRUCTURE.  Run here (the container that has /root/reference):
    make -C oracle ref && python oracle/gen_script_fuzz.py
The scripts are mutations of valid GEMM / pre-op schedules (wrong scopes,
missing or extra splits, bad extents, stage counts 0..5, primitive order
swaps, inline before/after pipelining, unknown primitives, syntax errors) so
most of them reach deep into the rule checks.
"""
import json
import os
import random
import subprocess
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
DRIVER = os.path.join(HERE, "_ref", "ref_driver")
OUT = os.path.join(ROOT, "tests", "golden", "scripts_fuzz.jsonl")


def divisors(n):
    return [d for d in range(1, n + 1) if n % d == 0]


def split_line(rng, M, N, K, tensor="C"):
    """A valid split of every dimension, then (one script in four) one mutation."""
    dims = []
    for size, names in ((M, ("i0", "i1")), (N, ("j0", "j1")), (K, ("ko", "ki"))):
        a = rng.choice(divisors(size))
        if rng.random() < 0.12:
            dims.append([(names[0], size)])  # one split
        else:
            dims.append([(names[0], a), (names[1], size // a)])
    mut = rng.random()
    if mut < 0.25:
        d = rng.randrange(3)
        kind = rng.randrange(7)
        name, ext = dims[d][-1]
        if kind == 0:
            dims[d][-1] = (name, ext + 1)                      # NonDivisibleSplit
        elif kind == 1:
            dims[d] = []                                      # missing dimension
        elif kind == 2:
            dims[d].append((name[0] + "2", 1))                # three splits
        elif kind == 3:
            dims[d][0] = ("x" + dims[d][0][0][1:], dims[d][0][1])  # bad name
        elif kind == 4:
            dims[d][0] = (dims[d][0][0], 0)                   # zero extent
        elif kind == 5:
            dims[d][-1] = (name, "q")                         # not an integer
        else:
            tensor = rng.choice(["A", "S2", "Z"])             # not the output
    parts = ["%s=%s" % kv for dim in dims for kv in dim]
    if rng.random() < 0.1:
        rng.shuffle(parts)
    return "tile %s %s" % (tensor, " ".join(parts))


def one_script(rng, preop):
    M = rng.choice([32, 64, 96, 128])
    N = rng.choice([32, 64, 128])
    K = rng.choice([16, 32, 64, 128])
    batch = rng.choice([1, 1, 1, 2, 3])
    a = "S2" if preop else "A"
    lines = []
    srcs = [a, "B"]
    shared = [t for t in srcs if rng.random() < 0.9]
    for t in shared:
        lines.append("cache_read %s shared" % t)
    regs = [t for t in shared if rng.random() < 0.5]
    for t in regs:
        lines.append("cache_read %s_shared register" % t)
    if rng.random() < 0.06:
        lines.append("cache_read %s %s" % (rng.choice(srcs + ["A_shared", "C", "Q"]),
                                           rng.choice(["shared", "register", "local", "global"])))
    lines.append(split_line(rng, M, N, K))
    bufs = ["%s_shared" % t for t in shared] + ["%s_reg" % t for t in regs]
    hints = []
    for b in bufs:
        if rng.random() < 0.8:
            hints.append("pipeline %s %d" % (b, rng.choice([2, 2, 3, 3, 4, 5] * 6 + [0, 1])))
    if rng.random() < 0.08:
        hints.append("pipeline %s %d" % (rng.choice(["A", "B", "C", "A_reg", "S2_shared", "B_shared"]),
                                         rng.choice([2, 3])))
    lines += hints
    if preop and rng.random() < 0.7:
        pos = len(lines) if rng.random() < 0.7 else rng.randrange(len(lines) + 1)
        lines.insert(pos, "inline %s" % ("S2" if rng.random() < 0.9 else rng.choice(["C", "A", "B"])))
    r = rng.random()
    if r < 0.08 and len(lines) > 1:  # order swap
        i = rng.randrange(len(lines) - 1)
        lines[i], lines[i + 1] = lines[i + 1], lines[i]
    elif r < 0.11:
        lines.insert(rng.randrange(len(lines) + 1), rng.choice(["vectorize C", "pipeline A_shared", "tile",
                                                                "cache_read A", "inline", "# note", "   "]))
    elif r < 0.13 and lines:
        del lines[rng.randrange(len(lines))]
    return M, N, K, batch, "\n".join(lines) + "\n"


def main(count=600, seed=20261017):
    if not os.path.exists(DRIVER):
        sys.exit("build the reference driver first: make -C oracle ref")
    rng = random.Random(seed)
    out = []
    with tempfile.TemporaryDirectory() as tmp:
        for i in range(count):
            preop = 1 if rng.random() < 0.3 else 0
            M, N, K, batch, text = one_script(rng, preop)
            p = os.path.join(tmp, "s.txt")
            with open(p, "w") as f:
                f.write(text)
            cmd = [DRIVER, "script", "--M", str(M), "--N", str(N), "--K", str(K), "--batch", str(batch),
                   "--script", p] + (["--preop", "1"] if preop else [])
            r = subprocess.run(cmd, capture_output=True, text=True, check=True)
            res = json.loads(r.stdout)
            out.append({"name": "fuzz_%03d" % i, "M": M, "N": N, "K": K, "batch": batch, "preop": preop,
                        "script": text, "result": res})
    with open(OUT, "w") as f:
        for o in out:
            f.write(json.dumps(o) + "\n")
    import collections
    print(collections.Counter((o["result"]["ok"], o["result"].get("rule") or o["result"].get("class"))
                              for o in out))


if __name__ == "__main__":
    main()
