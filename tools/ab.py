"""A/B kernel timing: build variant libraries from alternative beam_kernel.cu files and time them
back to back on the same GPU (tools/ablate.py-style CUDA-event timing, L2 flushed per decode).

  python tools/ab.py build NAME path/to/beam_kernel.cu      (here: nvcc, writes ab/libNAME.so)
  python tools/ab.py buildtree NAME path/to/csrc_dir          (a whole alternative csrc/ tree)
  python tools/ab.py time --workload c4 NAME[:ENV=VAL] ...   (on the GPU box)
"""
from __future__ import annotations

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def build(name, beam_src, csrc=None):
    sys.path.insert(0, os.path.join(ROOT, "paper_2508_07315_b200"))
    import build as B  # noqa: E402  (the package's build module, without importing the package)
    out = os.path.join(ROOT, "ab")
    os.makedirs(os.path.join(out, name), exist_ok=True)
    objs = []
    for src in B.sources():
        if csrc:
            s = os.path.join(os.path.abspath(csrc), os.path.basename(src))
        else:
            s = os.path.abspath(beam_src) if os.path.basename(src) == "beam_kernel.cu" else src
        obj = os.path.join(out, name, os.path.basename(src) + ".o")
        cmd = [B.NVCC, *B.ARCH, "-lineinfo", "-O3", "-std=c++17", "-fmad=false", "-Xcompiler", "-fPIC",
               "-Xcompiler", "-ffp-contract=off", "-I", B.INCLUDE, "-I", os.path.abspath(csrc) if csrc else B.CSRC,
               "-c", s, "-o", obj]
        subprocess.check_call(cmd)
        objs.append(obj)
    lib = os.path.join(out, f"lib{name}.so")
    subprocess.check_call([B.NVCC, *B.ARCH, "-shared", "-cudart", "static", "-o", lib, *objs])
    print(lib)


def time_all(workload, names, rounds=3, steps=20):
    res = {n: [] for n in names}
    for _ in range(rounds):
        for n in names:
            lib, *kv = n.split(":")
            env = dict(os.environ, FLEXCTC_LIB_AB=os.path.join(ROOT, "ab", f"lib{lib}.so"))
            for x in kv:
                k, v = x.split("=")
                env[k] = v
            out = subprocess.check_output([sys.executable, os.path.join(ROOT, "tools", "ablate.py"), "--workload",
                                           workload, "--steps", str(steps), "--only", "baseline"], env=env)
            res[n].append(json.loads(out.decode().strip().splitlines()[-1])["ms"])
    for n in names:
        print(json.dumps({"variant": n, "workload": workload, "ms": res[n], "min_ms": min(res[n])}))


if __name__ == "__main__":
    if sys.argv[1] == "build":
        build(sys.argv[2], sys.argv[3])
    elif sys.argv[1] == "buildtree":
        build(sys.argv[2], None, sys.argv[3])
    else:
        args = sys.argv[2:]
        wl = "c4"
        if args[0] == "--workload":
            wl, args = args[1], args[2:]
        time_all(wl, args)
