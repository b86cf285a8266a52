"""Build an experimental variant of the library with extra nvcc defines:
    python tools/build_variant.py NAME -DFOO=1 ...   -> build/variants/libgmt_b200_NAME.so
Load it with GMT_B200_LIB=build/variants/libgmt_b200_NAME.so."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1705_02403_b200 import build as B  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
obj = os.path.join(ROOT, "build", "variants", name)
os.makedirs(obj, exist_ok=True)
objs, procs = [], []
# ONLY=solve.cu,...: compile just those with the defines, link the in-tree
# build's objects (build/obj, current) for the rest
only = [x for x in os.environ.get("ONLY", "").split(",") if x]
for src in B.SOURCES:  # (in parallel)
    if only and src not in only:
        objs.append(os.path.join(B.OBJ, os.path.splitext(src)[0] + ".o"))
        continue
    o = os.path.join(obj, os.path.splitext(src)[0] + ".o")
    procs.append(subprocess.Popen([B.NVCC, *B.FLAGS, *defs, "-c", os.path.join(B.CSRC, src), "-o", o]))
    objs.append(o)
if any(p.wait() for p in procs):
    sys.exit("nvcc failed")
lib = os.path.join(ROOT, "build", "variants", f"libgmt_b200_{name}.so")
subprocess.run([B.NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", lib, *objs,
                "-cudart", "static"], check=True)
print(lib)
