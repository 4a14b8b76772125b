"""Builds libalcop.so (sm_100a kernels + C-ABI host code) in-tree with nvcc.

Used by __graft_entry__.build() and by `python -m paper_2210_16691_b200._build`.
The .so is git-ignored but travels to the GPU box with the gpurun snapshot.
"""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
LIB = os.environ.get("ALCOP_BUILD_LIB", os.path.join(HERE, "libalcop.so"))
EXTRA = os.environ.get("ALCOP_NVCC_EXTRA", "").split()
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CU_SOURCES = ["gemm_sm100.cu", "chain_sm100.cu", "stem_sm100.cu"]
CPP_SOURCES = ["alcop_api.cpp", "schedule.cpp", "model.cpp", "ir_frontend.cpp", "tuner.cpp", "sim.cpp",
               "sharded.cpp"]


def _sources():
    return [os.path.join(CSRC, f) for f in CU_SOURCES + CPP_SOURCES]


def _deps():
    deps = _sources() + [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))]
    deps.append(os.path.join(ROOT, "include", "alcop.h"))
    return deps


def up_to_date():
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(d) <= t for d in _deps())


def build(force=False, verbose=False):
    if not force and up_to_date():
        return LIB
    objdir = os.path.join(HERE, "_obj" + ("_" + os.path.basename(LIB) if "ALCOP_BUILD_LIB" in os.environ else ""))
    os.makedirs(objdir, exist_ok=True)
    objs = []
    common = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-O3", "-I" + os.path.join(ROOT, "include")] + EXTRA
    headers = [d for d in _deps() if d.endswith((".h", ".cuh"))]
    newest_header = max(os.path.getmtime(h) for h in headers)

    def fresh(src, o):  # per-object rebuild: the object is newer than its source and every header
        return (not force and os.path.exists(o) and os.path.getmtime(o) >= os.path.getmtime(src)
                and os.path.getmtime(o) >= newest_header)

    for f in CU_SOURCES:
        o = os.path.join(objdir, f + ".o")
        objs.append(o)
        if fresh(os.path.join(CSRC, f), o):
            continue
        cmd = [NVCC, *ARCH, *common, "-Xptxas", "-v" if verbose else "-O3", "-c", os.path.join(CSRC, f), "-o", o]
        subprocess.run(cmd, check=True)
    for f in CPP_SOURCES:
        o = os.path.join(objdir, f + ".o")
        objs.append(o)
        if fresh(os.path.join(CSRC, f), o):
            continue
        cmd = [NVCC, *ARCH, *common, "-x", "c++", "-c", os.path.join(CSRC, f), "-o", o]
        subprocess.run(cmd, check=True)
    tmp = LIB + ".tmp"
    subprocess.run([NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-lcudart_static", "-ldl", "-lrt", "-lpthread"],
                   check=True)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
