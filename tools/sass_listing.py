"""SASS evidence for the production kernels (measurement tool): per kernel,
counts of the tcgen05 / TMA / mbarrier mnemonics and the MMA-issue and
TMA-issue loops.  python tools/sass_listing.py > profiles/sass_r01.txt"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2210_16691_b200", "libalcop.so")
WANT = ["alcop_pipelined_gemm_kernel<__nv_bfloat16, 64, true, false, 0, false>",
        "alcop_pipelined_gemm_pair_kernel<__nv_bfloat16, 64>",
        "alcop_pipelined_gemm_kernel<__nv_bfloat16, 64, true, false, 1, false>"]
KEYS = ("UTCHMMA", "UTCQMMA", "UTCBAR", "LDTM", "UTMALDG", "UTMASTG", "UTMAPF", "SYNCS", "UTCATOMSWS", "ELECT",
        "FENCE", "ACQBULK")


def main():
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    funcs = re.split(r"\n\s*Function : ", sass)[1:]
    print("# SASS of the production kernels (sm_100a, cuobjdump -sass %s)" % os.path.relpath(LIB, ROOT))
    print("# UTCHMMA = tcgen05.mma, UTCBAR = tcgen05.commit, LDTM = tcgen05.ld, UTMALDG/UTMASTG = TMA load/store,")
    print("# SYNCS.* = mbarrier ops (PHASECHK.TRYWAIT = wait, ARRIVE.TRANS64 = arrive.expect_tx), UTCATOMSWS = TMEM alloc")
    for f in funcs:
        mangled = f.split("\n", 1)[0].strip()
        name = subprocess.run(["c++filt", mangled], capture_output=True, text=True).stdout.strip()
        hit = [w for w in WANT if w in name]
        if not hit:
            continue
        ins = [re.sub(r"/\* 0x[0-9a-f]+ \*/", "", l).strip() for l in f.split("\n")]
        ins = [l for l in ins if re.match(r"^/\*[0-9a-f]{4}\*/", l)]
        cnt = collections.Counter()
        for l in ins:
            op = l.split("*/", 1)[1].strip().split()
            if not op:
                continue
            m = op[0] if not op[0].startswith("@") else op[1]
            if m.startswith(KEYS):
                cnt[m.rstrip(";")] += 1
        print("\n## %s\n# %d instructions; key mnemonics:" % (name, len(ins)))
        for k, v in sorted(cnt.items()):
            print("   %5d %s" % (v, k))
        for key, title in (("UTCHMMA", "MMA issue (tcgen05.mma k-steps, then tcgen05.commit -> empty[slot])"),
                           ("UTMALDG", "TMA issue (producer_commit: arrive.expect_tx + bulk-tensor loads)")):
            idx = [i for i, l in enumerate(ins) if key in l]
            if not idx:
                continue
            lo, hi = max(0, idx[0] - 6), min(len(ins), idx[0] + 14)
            print("# %s:" % title)
            for l in ins[lo:hi]:
                print("   " + l)


if __name__ == "__main__":
    main()
