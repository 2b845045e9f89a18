"""In-tree build of the sm_100a engine: csrc/*.cu -> paper_1805_00569_b200/libpkrr_gpu.so.

Plain nvcc (no torch extension machinery): the library is a C-ABI shared object
(include/pkrr_gpu.h) with the CUDA runtime linked statically, so it loads the
same way from Python (ctypes), C++ (include/pkrr_gpu.hpp) or any FFI.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libpkrr_gpu.so")
SOURCES = ["kernels.cu", "engine.cu", "multi.cu", "dist.cu"]
HEADERS = sorted(f for f in os.listdir(CSRC) if f.endswith(".cuh"))
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC", "-Xcompiler", "-O3", "-Xptxas", "-O3"]


def _newer(target: str, deps) -> bool:
    if not os.path.exists(target):
        return False
    t = os.path.getmtime(target)
    return all(os.path.getmtime(p) <= t for p in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "pkrr_gpu.h")]
    if not force and _newer(LIB, deps):
        return LIB
    objs = []
    procs = []
    for src in SOURCES:
        obj = os.path.join(CSRC, src.replace(".cu", ".o"))
        extra = os.environ.get("PKRR_NVCC_DEFS", "").split()  # debug builds only
        cmd = ["nvcc", *NVCC_FLAGS, *extra, "-c", os.path.join(CSRC, src), "-o", obj]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        procs.append(subprocess.Popen(cmd))
        objs.append(obj)
    for p in procs:
        if p.wait() != 0:
            raise RuntimeError("nvcc failed")
    cmd = ["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", LIB, *objs]
    subprocess.run(cmd, check=True)
    for o in objs:
        os.remove(o)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
