"""SASS evidence for the kernels in libalcop.so (measurement tool).

For every kernel: instruction count and counts of the tcgen05 / TMA / mbarrier
mnemonics; for the production instantiations the bench times, the MMA-issue and
TMA-issue sequences.  Exits non-zero (and writes nothing useful) if the
library has no kernels or a production kernel lacks UTCHMMA / UTMALDG / LDTM —
a listing that is only a header is a failure, not evidence.

    python tools/sass_listing.py > profiles/sass_r02.txt
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2210_16691_b200", "libalcop.so")
# (substring of the demangled name, what the bench runs it for)
PRODUCTION = [
    ("alcop_pipelined_gemm_pair_kernel<__nv_bfloat16, 32, false, false, true, false>",
     "CTA-pair GEMM, 256 x 512 tile (two N = 256 MMAs per k-step): the C5 squares (headline)"),
    ("alcop_pipelined_gemm_pair_kernel<__nv_bfloat16, 64, false, false, false, false>",
     "CTA-pair GEMM (cta_group::2): BERT QKV / FFN1 / FFN2"),
    ("alcop_pipelined_gemm_pair_kernel<__nv_bfloat16, 64, false, false, false, true>",
     "CTA-pair implicit-GEMM conv (im2col loads, cta_group::2): ResNet-50 l3 / l4 layers"),
    ("alcop_pipelined_gemm_kernel<__nv_bfloat16, 64, true, false, 0, false, 4>",
     "single-CTA GEMM: BERT FFN2 / O, attention PV, config-1 class"),
    ("alcop_pipelined_gemm_kernel<__nv_bfloat16, 64, true, false, 0, false, 8>",
     "single-CTA GEMM, 8 epilogue warps: attention QK^T (K = 64)"),
    ("alcop_pipelined_gemm_kernel<__nv_bfloat16, 64, true, false, 1, false, 4>",
     "implicit-GEMM conv, TMA im2col (C % 64 == 0)"),
    ("alcop_pipelined_gemm_kernel<__nv_bfloat16, 64, true, false, 2, false, 4>",
     "implicit-GEMM conv, 8-channel im2col boxes (small C)"),
    ("alcop_pipelined_gemm_kernel<__nv_bfloat16, 64, true, false, 3, false, 4>",
     "implicit-GEMM conv, stem (ResNet-50 conv1, halo-padded NHWC8)"),
    ("alcop_chain_gemm_kernel<__nv_bfloat16, 64, false>", "several GEMMs in one persistent launch (alcop_gemm_chain)"),
    ("alcop_chain_gemm_kernel<__nv_bfloat16, 64, true>", "alcop_gemm_chain on CTA pairs (the BERT layer as one launch)"),
    ("alcop_stem_conv_kernel<__nv_bfloat16, 3, 7, 2, false>",
     "resident-filter conv, pixel pairs, four output rows per tile: the ResNet-50 stem (C = 4, 7x7/2)"),
    ("alcop_stem_conv_kernel<__nv_bfloat16, 0, 7, 2, false>",
     "resident-filter conv, pixel-pair mode, one output row per tile (other C = 4 stride-2 shapes)"),
    ("alcop_stem_conv_kernel<__nv_bfloat16, 1, 3, 3, false>",
     "resident-filter conv, window mode: 3x3 stride-1 C = 64 (ResNet-50 l1 3x3)"),
    ("alcop_stem_conv_kernel<__nv_bfloat16, 2, 0, 0, false>",
     "window conv with a streamed filter (separate A / B rings): C > 64, K <= 128"),
    ("alcop_stem_conv_kernel<__nv_bfloat16, 1, 3, 3, true>",
     "window conv on CTA pairs (cta_group::2, M = 256): ResNet-50 l1 3x3"),
    ("alcop_stem_conv_kernel<__nv_bfloat16, 2, 0, 0, true>",
     "window conv, streamed filter, on CTA pairs: ResNet-50 l2 3x3"),
]
KEYS = ("UTCHMMA", "UTCQMMA", "UTCBAR", "LDTM", "UTMALDG", "UTMASTG", "UTMAPF", "UTMACMDFLUSH", "SYNCS", "UTCATOMSWS",
        "UTCBAR", "ELECT", "FENCE", "ACQBULK", "MEMBAR")
REQUIRED = ("UTCHMMA", "UTMALDG", "LDTM")


def kernels(sass):
    for f in re.split(r"\n\s*Function : ", sass)[1:]:
        mangled = f.split("\n", 1)[0].strip()
        name = subprocess.run(["c++filt", mangled], capture_output=True, text=True).stdout.strip()
        ins = [re.sub(r"/\* 0x[0-9a-f]+ \*/", "", l).strip() for l in f.split("\n")]
        ins = [l for l in ins if re.match(r"^/\*[0-9a-f]{4}\*/", l)]
        yield name, ins


def mnemonic(line):
    op = line.split("*/", 1)[1].strip().split()
    if not op:
        return ""
    return (op[1] if op[0].startswith("@") and len(op) > 1 else op[0]).rstrip(";")


def main():
    if not os.path.exists(LIB):
        sys.exit("sass_listing: %s not built" % LIB)
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True, check=True).stdout
    rows = []
    prod = {}
    for name, ins in kernels(sass):
        cnt = collections.Counter(m for m in map(mnemonic, ins) if m.startswith(KEYS))
        short = re.sub(r"alcop::\(anonymous namespace\)::", "", name.split("(CUtensorMap")[0].split("(alcop::")[0])
        rows.append((short, len(ins), cnt))
        for key, why in PRODUCTION:
            if key in name:
                prod[key] = (why, name, ins, cnt)
    if not rows:
        sys.exit("sass_listing: no kernels in %s" % LIB)
    missing = [k for k, _ in PRODUCTION if k not in prod]
    weak = [k for k, (_, _, _, c) in prod.items() if not all(any(m.startswith(r) for m in c) for r in REQUIRED)]
    if missing or weak:
        sys.exit("sass_listing: production kernels missing %s / without %s: %s" % (missing, REQUIRED, weak))
    print("# SASS of libalcop.so (sm_100a; cuobjdump -sass %s), %d kernels" % (os.path.relpath(LIB, ROOT), len(rows)))
    print("# UTCHMMA = tcgen05.mma (kind::f16), UTCBAR = tcgen05.commit -> mbarrier, LDTM = tcgen05.ld,")
    print("# UTMALDG / UTMASTG = TMA bulk-tensor load / store (.IM2COL = im2col mode, .2CTA = cta_group::2),")
    print("# SYNCS.* = mbarrier ops (PHASECHK.TRANS64.TRYWAIT = try_wait.parity, ARRIVE.TRANS64 = arrive[.expect_tx]),")
    print("# UTCATOMSWS = tcgen05.alloc / dealloc (TMEM)")
    cols = ["UTCHMMA", "UTCBAR", "LDTM", "UTMALDG", "UTMASTG", "SYNCS"]
    print("\n## Per-kernel mnemonic counts (prefix match)\n%-96s %6s " % ("kernel", "instr") +
          " ".join("%8s" % c for c in cols))
    tot = collections.Counter()
    for short, n, cnt in sorted(rows):
        agg = {c: sum(v for k, v in cnt.items() if k.startswith(c)) for c in cols}
        tot.update(agg)
        print("%-96s %6d " % (short[:96], n) + " ".join("%8d" % agg[c] for c in cols))
    print("%-96s %6s " % ("TOTAL", "") + " ".join("%8d" % tot[c] for c in cols))
    for key, _ in PRODUCTION:
        why, name, ins, cnt = prod[key]
        print("\n## %s\n# %s\n# %d instructions; key mnemonics:" % (key, why, len(ins)))
        for k, v in sorted(cnt.items()):
            print("   %5d %s" % (v, k))
        for mark, title in (("UTCHMMA", "MMA issue: tcgen05.mma k-steps of one chunk, then tcgen05.commit -> empty[slot]"),
                            ("UTMALDG", "TMA issue: producer_commit = arrive.expect_tx + bulk-tensor loads"),
                            ("LDTM", "epilogue: tcgen05.ld of the TMEM accumulator")):
            idx = [i for i, l in enumerate(ins) if mark in l]
            if not idx:
                continue
            lo, hi = max(0, idx[0] - 6), min(len(ins), idx[0] + 14)
            print("# %s:" % title)
            for l in ins[lo:hi]:
                print("   " + l)


if __name__ == "__main__":
    main()
