"""Builds libflexctc.so (the C-ABI library) in-tree with nvcc for sm_100a.

nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -fmad=false (explicit __fmaf_rn
only: reading R19), static cudart, -fPIC shared library. Host C++ builders are compiled by
the same nvcc invocation (g++ backend, -ffp-contract=off)."""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libflexctc.so")
# the per-phase cycle counters (-DFLEXCTC_PHASE_TIMERS) go to their own library, so a timers build
# never replaces the product library (and FLEXCTC_PHASE_TIMERS=1 selects it at import)
LIB_TIMERS = os.path.join(HERE, "libflexctc_timers.so")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def deps():
    return sources() + glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(INCLUDE, "*.h"))


def lib_path(timers: bool | None = None) -> str:
    if timers is None:
        timers = os.environ.get("FLEXCTC_PHASE_TIMERS") == "1"
    return LIB_TIMERS if timers else LIB


def up_to_date(timers: bool | None = None) -> bool:
    lib = lib_path(timers)
    if not os.path.exists(lib):
        return False
    t = os.path.getmtime(lib)
    return all(os.path.getmtime(d) <= t for d in deps())


def build(force: bool = False, verbose: bool = False, timers: bool | None = None) -> str:
    """timers: compile the per-phase cycle counters in (-DFLEXCTC_PHASE_TIMERS; also via the
    FLEXCTC_PHASE_TIMERS=1 environment variable)."""
    if timers is None:
        timers = os.environ.get("FLEXCTC_PHASE_TIMERS") == "1"
    lib = lib_path(timers)
    if not force and up_to_date(timers):
        return lib
    objdir = os.path.join(HERE, "build_timers" if timers else "build")
    os.makedirs(objdir, exist_ok=True)
    objs = []
    for src in sources():
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        cmd = [NVCC, *ARCH, "-lineinfo", "-O3", "-std=c++17", "-fmad=false", "-Xcompiler", "-fPIC",
               "-Xcompiler", "-ffp-contract=off", "-I", INCLUDE, "-I", CSRC, "-c", src, "-o", obj]
        if src.endswith(".cu"):
            cmd += ["-Xptxas", "-v"] if verbose else []
            cmd += ["-DFLEXCTC_PHASE_TIMERS"] if timers else []
        subprocess.check_call(cmd)
        objs.append(obj)
    tmp = lib + f".tmp{os.getpid()}"
    subprocess.check_call([NVCC, *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs])
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, timers=True if "--timers" in sys.argv else None))
