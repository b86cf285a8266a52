"""Build the B200 library in-tree: libgmt_b200.so (sm_100a only).

    python -m paper_1705_02403_b200.build

Every .cu under csrc/ is compiled with
  -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false
(--fmad=false: no FMA contraction anywhere, the reference's x86-64 double
semantics) and linked into one shared object next to this
file, so it travels to the GPU box with the repo snapshot.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libgmt_b200.so")
OBJ = os.path.join(ROOT, "build", "obj")
SOURCES = ["solve.cu", "graph.cu", "di_graph.cu", "sample.cu", "capi.cu", "cache.cu", "sim.cu", "batch_build.cu", "pool.cu",
           "problem_file.cpp"]
HEADERS = ["common.cuh", "solve.cuh", "internal.cuh", "offline.cuh", "di.cuh", "quad.cuh", "dubins.cuh",
           "sample_dev.cuh"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "--fmad=false",
         "-std=c++17", "-Xcompiler", "-fPIC", "-I" + os.path.join(ROOT, "include"),
         "-I" + CSRC]


def _newer(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, force: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    hdrs = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(ROOT, "include", "gmt_b200.h")]
    objs = []
    procs = []
    for src in SOURCES:  # translation units compile in parallel
        s = os.path.join(CSRC, src)
        o = os.path.join(OBJ, os.path.splitext(src)[0] + ".o")
        objs.append(o)
        if force or _newer(o, [s] + hdrs):
            cmd = [NVCC, *FLAGS, "-c", s, "-o", o]
            if verbose:
                print(" ".join(cmd), flush=True)
            procs.append((src, subprocess.Popen(cmd)))
    failed = [src for src, p in procs if p.wait() != 0]
    if failed:
        raise subprocess.CalledProcessError(1, "nvcc " + " ".join(failed))
    if force or _newer(LIB, objs):
        cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", LIB, *objs,
               "-cudart", "static"]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
    return LIB


if __name__ == "__main__":
    build(verbose=True, force="--force" in sys.argv)
