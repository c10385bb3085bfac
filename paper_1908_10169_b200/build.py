"""Build libbilu.so in-tree: nvcc for the sm_100a kernels, g++ for the host
orchestrator, linked into one shared library with a C ABI (include/bilu.h)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libbilu.so")
LIB_PROF = os.path.join(HERE, "libbilu_prof.so")   # diagnostic build with per-phase clock64 counters
LIB_TUNE = os.path.join(HERE, "libbilu_tune.so")   # tools/ build that reads the BILU_* tuning switches
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CU_SOURCES = ["bilu_factor.cu", "bilu_merge.cu", "bilu_apply.cu", "bilu_util.cu", "bilu_krylov.cu", "bilu_blocking.cu",
              "bilu_matching.cu"]
CPP_SOURCES = ["bilu_host.cpp"]
HEADERS = ["bilu_internal.h", "dgemm_cta.cuh", os.path.join("..", "..", "include", "bilu.h")]


def _newest_source() -> float:
    paths = [os.path.join(CSRC, f) for f in CU_SOURCES + CPP_SOURCES + HEADERS] + [__file__]
    return max(os.path.getmtime(p) for p in paths)


def build(force: bool = False, verbose: bool = False, profile: bool = False, defines=(), out=None,
          tuning: bool = False) -> str:
    """Compile and link libbilu.so (or a variant: `defines` extra -D flags, `out` library path;
    `tuning`: libbilu_tune.so, which reads the BILU_* tuning/diagnostic environment switches)."""
    if tuning:
        defines, out = tuple(defines) + ("BILU_TUNING",), out or LIB_TUNE
    lib = out or (LIB_PROF if profile else LIB)
    if not force and os.path.exists(lib) and os.path.getmtime(lib) >= _newest_source():
        return lib
    objdir = os.path.join(HERE, "build_prof" if profile else "build")
    if out:
        objdir = os.path.join(HERE, "build_" + os.path.basename(out).replace(".so", ""))
    os.makedirs(objdir, exist_ok=True)
    objs = []
    hdr_time = max(os.path.getmtime(os.path.join(CSRC, h)) for h in HEADERS + []) if HEADERS else 0.0
    hdr_time = max(hdr_time, os.path.getmtime(__file__))

    def fresh(src, o):   # incremental: an object newer than its source and every header is kept
        return (not force and os.path.exists(o) and
                os.path.getmtime(o) >= max(os.path.getmtime(src), hdr_time))

    for f in CU_SOURCES:
        o = os.path.join(objdir, f + ".o")
        objs.append(o)
        if fresh(os.path.join(CSRC, f), o):
            continue
        cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
               "-I", os.path.join(ROOT, "include"), "-c", os.path.join(CSRC, f), "-o", o]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        if profile:
            cmd.insert(1, "-DBILU_PROFILE")
        for d in defines:
            cmd.insert(1, "-D" + d)
        subprocess.check_call(cmd)
    for f in CPP_SOURCES:
        o = os.path.join(objdir, f + ".o")
        objs.append(o)
        if fresh(os.path.join(CSRC, f), o):
            continue
        subprocess.check_call(["g++", "-std=c++17", "-O2", "-fPIC", "-Wall", "-I/usr/local/cuda/include",
                               "-I", os.path.join(ROOT, "include"), "-c", os.path.join(CSRC, f), "-o", o])
    tmp = lib + ".tmp%d" % os.getpid()
    subprocess.check_call([NVCC, *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs])
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    defs = [a[2:] for a in sys.argv[1:] if a.startswith("-D")]
    outs = [a[6:] for a in sys.argv[1:] if a.startswith("--out=")]
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, profile="--profile" in sys.argv,
                defines=defs, out=os.path.join(HERE, outs[0]) if outs else None, tuning="--tuning" in sys.argv))
