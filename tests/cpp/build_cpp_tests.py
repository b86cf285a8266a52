"""Build tests/cpp/test_shim (the C++ drop-in test) against the in-tree
libgmt_b200.so and the oracle's liboracle.so.  Called by
__graft_entry__.build(); the binary lands in build/ and travels with the repo
snapshot to the GPU box."""
from __future__ import annotations

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
OUT = os.path.join(ROOT, "build", "test_shim")


def build(verbose: bool = False) -> str:
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    pkg = os.path.join(ROOT, "paper_1705_02403_b200")
    orc = os.path.join(ROOT, "oracle")
    cmd = ["g++", "-std=c++20", "-O2", "-Wall", "-Wextra", "-I" + os.path.join(ROOT, "include"),
           os.path.join(HERE, "test_shim.cpp"), "-o", OUT,
           os.path.join(pkg, "libgmt_b200.so"), os.path.join(orc, "liboracle.so"),
           "-Wl,-rpath," + pkg, "-Wl,-rpath," + orc, "-Wl,-rpath,$ORIGIN/../paper_1705_02403_b200",
           "-Wl,-rpath,$ORIGIN/../oracle"]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    return OUT


if __name__ == "__main__":
    build(verbose=True)
